"""CLI (paper_1411_5283_b200/cli.py): exit codes and the host-side order check
on CPU; sort / clean / verify / bench through the GPU against the oracle on a GPU box."""
import random

import numpy as np
import pytest

import oracle
from paper_1411_5283_b200 import cli


def _text(seed, n=20000):
    rng = random.Random(seed)
    words = [bytes(rng.choice(b"abcdeXYZ") for _ in range(rng.choice([1, 1, 2, 3, 5, 8, 13, 40])))
             for _ in range(n)]
    seps = [rng.choice([b" ", b", ", b"\n", b"--", b"'"]) for _ in range(n)]
    return b"".join(w + s for w, s in zip(words, seps))


# ---------------------------------------------------------------------------- CPU
def test_usage_errors_exit_1(capsys):
    assert cli.main([]) == cli.EXIT_USAGE
    assert cli.main(["frobnicate"]) == cli.EXIT_USAGE
    assert cli.main(["sort"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "x", "--algo", "nope"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "x", "--trials", "0"]) == cli.EXIT_USAGE


def test_unreadable_input_exit_2(tmp_path):
    missing = str(tmp_path / "missing.txt")
    for argv in (["sort", missing], ["clean", missing], ["verify", missing, missing], ["bench", missing]):
        assert cli.main(argv) == cli.EXIT_IO


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_order_check_accepts_oracle_output(seed):
    ref = oracle.sort(_text(seed, 3000))
    assert cli.first_order_violation(np.frombuffer(ref.words, np.uint8)) is None


def test_order_check_names_first_bad_line():
    def v(s):
        return cli.first_order_violation(np.frombuffer(s, np.uint8))

    assert v(b"") is None
    assert v(b"a\nb\nab\nba\n") is None
    assert v(b"a\na\nab\nab\n") is None                      # duplicates are fine
    assert v(b"b\na\n") == (2, "out of (length, alphabetical) order")
    assert v(b"a\nab\nb\n") == (3, "out of (length, alphabetical) order")   # length goes down
    assert v(b"a\nzz\nab\n") == (3, "out of (length, alphabetical) order")
    assert v(b"a\nB\n") == (2, "not a non-empty lower-case word")
    assert v(b"a\n\nb\n") == (2, "not a non-empty lower-case word")
    assert v(b"a\nb") == (2, "last line not terminated by a newline")
    # swapping two lines of a real sorted output is caught at the second one
    ref = oracle.sort(_text(5, 2000)).words.split(b"\n")[:-1]
    i = next(i for i in range(len(ref) - 1) if ref[i] != ref[i + 1] and len(ref[i]) == len(ref[i + 1]))
    ref[i], ref[i + 1] = ref[i + 1], ref[i]
    assert v(b"\n".join(ref) + b"\n") == (i + 2, "out of (length, alphabetical) order")


# ---------------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def built():
    import build_native

    build_native.build_wsort()


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["auto", "lsd_radix", "dense_msd"])
def test_sort_writes_oracle_output(built, tmp_path, algo):
    text = _text(11)
    inp, out = tmp_path / "in.txt", tmp_path / "out.txt"
    inp.write_bytes(text)
    assert cli.main(["sort", str(inp), "-o", str(out), "--algo", algo]) == cli.EXIT_OK
    assert out.read_bytes() == oracle.sort(text).words
    assert cli.main(["verify", str(inp), str(out)]) == cli.EXIT_OK


@pytest.mark.gpu
def test_clean_is_length_major_source_order(built, tmp_path, capsys):
    text = _text(12)
    inp, out = tmp_path / "in.txt", tmp_path / "clean.txt"
    inp.write_bytes(text)
    assert cli.main(["clean", str(inp), "-o", str(out)]) == cli.EXIT_OK
    pos, ln = oracle.tokenize(text)
    low = text.lower()
    order = sorted(range(len(pos)), key=lambda i: (int(ln[i]), i))
    want = b"".join(low[int(pos[i]): int(pos[i]) + int(ln[i])] + b"\n" for i in order)
    assert out.read_bytes() == want
    err = capsys.readouterr().err
    assert f"words {len(pos)}" in err


@pytest.mark.gpu
def test_verify_rejects_swap_deletion_and_foreign_word(built, tmp_path):
    text = _text(13)
    inp = tmp_path / "in.txt"
    inp.write_bytes(text)
    lines = oracle.sort(text).words.split(b"\n")[:-1]
    cases = {
        "deleted": lines[:100] + lines[101:],
        "extra": lines + [lines[-1]],          # still ordered, but one word too many
        "swapped": list(lines),
    }
    i = next(i for i in range(len(lines) - 1) if lines[i] != lines[i + 1] and len(lines[i]) == len(lines[i + 1]))
    cases["swapped"][i], cases["swapped"][i + 1] = cases["swapped"][i + 1], cases["swapped"][i]
    for name, ls in cases.items():
        f = tmp_path / f"{name}.txt"
        f.write_bytes(b"\n".join(ls) + b"\n")
        want = cli.EXIT_OK if ls == lines else cli.EXIT_VERIFY
        assert cli.main(["verify", str(inp), str(f)]) == want, name


@pytest.mark.gpu
def test_empty_file(built, tmp_path):
    inp, out = tmp_path / "empty.txt", tmp_path / "out.txt"
    inp.write_bytes(b"")
    assert cli.main(["sort", str(inp), "-o", str(out)]) == cli.EXIT_OK
    assert out.read_bytes() == b""
    assert cli.main(["verify", str(inp), str(out)]) == cli.EXIT_OK


@pytest.mark.gpu
def test_bench_csv(built, tmp_path):
    inp, out = tmp_path / "in.txt", tmp_path / "bench.csv"
    inp.write_bytes(_text(14))
    assert cli.main(["bench", str(inp), "--algo", "auto,lsd_radix", "--trials", "2", "--warmup", "1",
                     "--format", "csv", "-o", str(out)]) == cli.EXIT_OK
    rows = out.read_text().strip().split("\n")
    assert rows[0] == "algo,mean_time_s,words_per_s,bytes,trials"
    assert [r.split(",")[0] for r in rows[1:]] == ["auto", "lsd_radix"]
    assert all(float(r.split(",")[2]) > 0 for r in rows[1:])


@pytest.mark.gpu
@pytest.mark.parametrize("cmd", ["sort", "clean"])
def test_word_too_long_exit_2(tmp_path, cmd, capsys):
    """A run of > 255 letters (reading A7, WSORT_E_WORD_TOO_LONG): a one-line diagnostic and exit 2,
    not a traceback."""
    p = tmp_path / "blob.txt"
    p.write_bytes(b"hello " + b"Q" * 300 + b" world\n")
    assert cli.main([cmd, str(p), "-o", str(tmp_path / "out.txt")]) == cli.EXIT_IO
    assert "cannot process input" in capsys.readouterr().err
