"""wsort command line: clean / sort / verify / bench (interface after SPEC.md:357-424).

    python -m paper_1411_5283_b200.cli sort   INPUT [-o OUT] [--algo auto] [--device 0]
    python -m paper_1411_5283_b200.cli clean  INPUT [-o OUT]
    python -m paper_1411_5283_b200.cli verify INPUT SORTED
    python -m paper_1411_5283_b200.cli bench  INPUT [--trials 10] [--algo auto,...] [--format table|csv]

Every command runs the method on the GPU through the public API (api.WSort); there is no CPU path.
Output files hold one word per line, the library's own output format.

  sort    the sorted corpus: length-major, alphabetical within a length (§3 Pre-processing).
  clean   the words "after removing the special characters", lower-cased, grouped by
          length, original order within a length; bucket histogram on stderr.
  verify  exit 0 iff SORTED is (a) ordered by (length, word) and (b) the multiset of INPUT's words.
          (a) is checked on the host from SORTED alone; (b) against the GPU's canonical output (a sorted
          sequence is fixed by its multiset, so (a) + byte equality <=> (b)). Names the first bad line.
  bench   mean wall time of load+tokenize+sort+fetch per trial, one row per algorithm.

Exit codes: 0 ok, 1 usage error, 2 I/O error or an input the library refuses (e.g. a
run of more than 255 letters, WSORT_E_WORD_TOO_LONG; reading A7) or a library failure, 3 verification
failure. Diagnostics go to
stderr, data to stdout or --output.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_VERIFY = 0, 1, 2, 3


class _Usage(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _Usage(message)


def _read(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        return np.frombuffer(f.read(), dtype=np.uint8)


def _write(path: str | None, data) -> None:
    buf = memoryview(np.ascontiguousarray(data, dtype=np.uint8))
    if path is None or path == "-":
        sys.stdout.buffer.write(buf)
        sys.stdout.buffer.flush()
    else:
        with open(path, "wb") as f:
            f.write(buf)


def _run(text: np.ndarray, algo: str, device: int, src_off: bool = False):
    from .api import WSort

    with WSort(device) as ws:
        ws.load_text(text)
        ws.tokenize()
        ws.sort(algo, src_off=src_off)
        return ws.fetch(src_off=src_off)


def bucket_rows(words: np.ndarray, off: list, L: int) -> np.ndarray:
    """The words of length L as an (n_L, L+1) byte matrix (each row = word + '\\n')."""
    lo, hi = off[L], off[L + 1]
    if hi == lo:
        return np.empty((0, L + 1), np.uint8)
    base = sum((off[j + 1] - off[j]) * (j + 1) for j in range(1, L))
    return words[base: base + (hi - lo) * (L + 1)].reshape(hi - lo, L + 1)


def first_order_violation(sorted_bytes: np.ndarray) -> tuple[int, str] | None:
    """(1-based line, reason) of the first line of a one-word-per-line file that breaks the
    (length, then alphabetical) order or is not a lower-case word; None if there is none."""
    data = np.asarray(sorted_bytes, dtype=np.uint8)
    if data.size == 0:
        return None
    if data[-1] != 0x0A:
        return (int(np.count_nonzero(data == 0x0A)) + 1, "last line not terminated by a newline")
    nl = np.flatnonzero(data == 0x0A)
    starts = np.concatenate(([0], nl[:-1] + 1))
    lens = nl - starts
    body = np.ones(data.size, bool)
    body[nl] = False
    bad = np.flatnonzero(body & ((data < ord("a")) | (data > ord("z"))))
    bad_line = None
    if bad.size:
        bad_line = int(np.searchsorted(nl, bad[0]))
    if (lens == 0).any():
        z = int(np.flatnonzero(lens == 0)[0])
        bad_line = z if bad_line is None else min(bad_line, z)
    dec = np.flatnonzero(lens[1:] < lens[:-1])
    first = None if dec.size == 0 else int(dec[0]) + 1
    # within each length: rows of equal width compare as fixed-size byte strings
    for L in np.unique(lens):
        idx = np.flatnonzero(lens == L)
        if idx.size < 2 or L == 0:
            continue
        rows = data[(starts[idx][:, None] + np.arange(L)[None, :])].copy().view(f"S{L}").reshape(-1)
        down = np.flatnonzero(rows[1:] < rows[:-1])
        if down.size:
            cand = int(idx[down[0] + 1])
            first = cand if first is None else min(first, cand)
    if bad_line is not None and (first is None or bad_line <= first):
        return (bad_line + 1, "not a non-empty lower-case word")
    if first is not None:
        return (first + 1, "out of (length, alphabetical) order")
    return None


def cmd_sort(a) -> int:
    text = _read(a.input)
    words, off = _run(text, a.algo, a.device)
    _write(a.output, words)
    print(f"words {off[-1]}  max_len {len(off) - 2}", file=sys.stderr)
    return EXIT_OK


def cmd_clean(a) -> int:
    text = _read(a.input)
    words, off, src = _run(text, "lsd_radix", a.device, src_off=True)
    parts, hist = [], []
    for L in range(1, len(off) - 1):
        rows = bucket_rows(words, off, L)
        if rows.shape[0] == 0:
            continue
        order = np.argsort(src[off[L]: off[L + 1]], kind="stable")
        parts.append(rows[order].reshape(-1))
        hist.append(f"{L}:{rows.shape[0]}")
    _write(a.output, np.concatenate(parts) if parts else np.empty(0, np.uint8))
    print(f"words {off[-1]}", file=sys.stderr)
    print("buckets " + " ".join(hist), file=sys.stderr)
    return EXIT_OK


def cmd_verify(a) -> int:
    text = _read(a.input)
    got = _read(a.sorted)
    v = first_order_violation(got)
    if v is not None:
        print(f"verify: line {v[0]}: {v[1]}", file=sys.stderr)
        return EXIT_VERIFY
    want, off = _run(text, a.algo, a.device)
    if got.size == want.size and np.array_equal(got, want):
        print(f"verify: ok ({off[-1]} words)", file=sys.stderr)
        return EXIT_OK
    n = min(got.size, want.size)
    diff = np.flatnonzero(got[:n] != want[:n])
    pos = int(diff[0]) if diff.size else n
    line = int(np.count_nonzero(got[:pos] == 0x0A)) + 1
    print(f"verify: line {line}: not the word multiset of {a.input} "
          f"({int(np.count_nonzero(got == 0x0A))} lines vs {off[-1]} words)", file=sys.stderr)
    return EXIT_VERIFY


def cmd_bench(a) -> int:
    from .api import WSort

    text = _read(a.input)
    algos = [s for s in a.algo.split(",") if s]
    rows = []
    with WSort(a.device) as ws:
        for algo in algos:
            times = []
            n = 0
            for t in range(a.warmup + a.trials):
                t0 = time.perf_counter()
                ws.load_text(text)
                n = ws.tokenize()
                ws.sort(algo)
                ws.fetch()
                if t >= a.warmup:
                    times.append(time.perf_counter() - t0)
            mean = sum(times) / len(times)
            rows.append((algo, mean, n / mean, len(times)))
    if a.format == "csv":
        out = "algo,mean_time_s,words_per_s,bytes,trials\n" + "".join(
            f"{r[0]},{r[1]:.6f},{r[2]:.1f},{text.size},{r[3]}\n" for r in rows)
    else:
        out = f"{'algo':<12} {'mean_time_s':>12} {'words/s':>14} {'trials':>6}\n" + "".join(
            f"{r[0]:<12} {r[1]:>12.6f} {r[2]:>14.4g} {r[3]:>6}\n" for r in rows)
    _write(a.output, np.frombuffer(out.encode(), np.uint8))
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    from ._lib import ALGOS

    p = _Parser(prog="wsort", description="GPU word sort by (length, alphabetical) — arXiv 1411.5283")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    def common(sp, algo=True):
        sp.add_argument("--device", type=int, default=0)
        if algo:
            sp.add_argument("--algo", default="auto", choices=sorted(ALGOS))

    s = sub.add_parser("sort")
    s.add_argument("input")
    s.add_argument("-o", "--output")
    common(s)
    c = sub.add_parser("clean")
    c.add_argument("input")
    c.add_argument("-o", "--output")
    common(c, algo=False)
    v = sub.add_parser("verify")
    v.add_argument("input")
    v.add_argument("sorted")
    common(v)
    b = sub.add_parser("bench")
    b.add_argument("input")
    b.add_argument("-o", "--output")
    b.add_argument("--algo", default="auto")
    b.add_argument("--trials", type=int, default=10)
    b.add_argument("--warmup", type=int, default=2)
    b.add_argument("--format", default="table", choices=["table", "csv"])
    b.add_argument("--device", type=int, default=0)
    return p


def main(argv=None) -> int:
    try:
        a = build_parser().parse_args(argv)
        if a.cmd == "bench":
            from ._lib import ALGOS

            bad = [s for s in a.algo.split(",") if s not in ALGOS]
            if bad or a.trials < 1 or a.warmup < 0:
                raise _Usage(f"bad --algo {bad} or --trials/--warmup")
        for path in [getattr(a, "input", None), getattr(a, "sorted", None)]:
            if path is not None and not os.access(path, os.R_OK):
                print(f"wsort: cannot read {path}", file=sys.stderr)
                return EXIT_IO
        return {"sort": cmd_sort, "clean": cmd_clean, "verify": cmd_verify, "bench": cmd_bench}[a.cmd](a)
    except _Usage as e:
        print(f"wsort: usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except OSError as e:
        print(f"wsort: I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except Exception as e:   # the library refused the input or failed (WSortError: status + message)
        from .api import WSortError

        if not isinstance(e, WSortError):
            raise
        print(f"wsort: cannot process input: {e}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
