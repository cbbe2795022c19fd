"""Ingestion formats: the parsers of csrc/ingest.cpp against the
reference's rules and wording (proj/src/graph.cpp:68-109, 302-336;
proj/src/partition.cpp:458-493; the reference's own IO tests,
proj/tests/test_graph.cpp:11-37, 180-194, test_partition.cpp:188-199, also run
through the C++ drop-in in tests/test_reference_suites_gpu.py). No GPU."""
import numpy as np
import pytest

from paper_2407_14106_b200 import ingest
from paper_2407_14106_b200._lib import DataError


def test_edge_list_basics():
    n, s, d = ingest.parse_edge_list("0 1\n1 2\n# comment\n\n  2 0\n")
    assert n == 3 and s.tolist() == [0, 1, 2] and d.tolist() == [1, 2, 0]
    n, s, d = ingest.parse_edge_list("0 1\n", 5)
    assert n == 5
    n, s, d = ingest.parse_edge_list("", 4)  # hint: empty graph allowed
    assert n == 4 and s.size == 0


@pytest.mark.parametrize("text,hint,msg", [
    ("0 x\n", None, 'parse error at line 1: bad token "x"'),
    ("0 1\n2\n", None, 'parse error at line 2: expected "src dst"'),
    ("0 1 2\n", None, 'parse error at line 1: expected "src dst"'),
    ("# c\n0 -1\n", None, "range error at line 2: negative node id"),
    ("0 1\n0 3\n", 3, "range error at line 2: node id 3 >= hint 3"),
    ("# only comments\n\n", None, "empty graph"),
])
def test_edge_list_errors(text, hint, msg):
    with pytest.raises(DataError) as e:
        ingest.parse_edge_list(text, hint)
    assert msg in str(e.value)


def test_edge_list_parallel_chunks_and_line_numbers():
    """> 1 MiB parses on several threads: same edges as a sequential parse, and
    an error deep in the file reports its global line number."""
    rng = np.random.default_rng(0)
    m = 400000
    s, d = rng.integers(0, 10**6, m), rng.integers(0, 10**6, m)
    lines = [f"{a}\t{b}" for a, b in zip(s, d)]
    lines.insert(1234, "# a comment")
    text = "\n".join(lines) + "\n"
    n, gs, gd = ingest.parse_edge_list(text)
    assert n == max(s.max(), d.max()) + 1
    assert np.array_equal(gs, s) and np.array_equal(gd, d)
    bad = lines[:]
    bad[300000] = "7 oops"
    with pytest.raises(DataError, match='line 300001: bad token "oops"'):
        ingest.parse_edge_list("\n".join(bad) + "\n")


def test_gtf1_round_trip_and_errors():
    m = np.random.default_rng(1).standard_normal((5, 3)).astype(np.float32)
    b = ingest.encode_gtf1(m)
    assert b[:4] == b"GTF1" and len(b) == 20 + 5 * 3 * 4
    assert np.array_equal(ingest.decode_gtf1(b), m)
    with pytest.raises(DataError, match="bad magic"):
        ingest.decode_gtf1(b"GTF2" + b[4:])
    with pytest.raises(DataError, match="truncated header"):
        ingest.decode_gtf1(b[:10])
    with pytest.raises(DataError, match="truncated at row 4"):
        ingest.decode_gtf1(b[:-4])


def test_permutation_text():
    fw = np.array([2, 0, 3, 1])
    text = ingest.format_permutation(fw)
    assert text == "0 2\n1 0\n2 3\n3 1\n"
    f, i = ingest.parse_permutation("# header\n" + text)
    assert np.array_equal(f, fw) and np.array_equal(i, np.argsort(fw))
    with pytest.raises(DataError, match="permutation: parse error at line 1"):
        ingest.parse_permutation("0 x\n")
    with pytest.raises(DataError, match="permutation: invalid pair 0 5"):
        ingest.parse_permutation("0 5\n1 0\n")
    with pytest.raises(DataError, match="permutation: invalid pair 0 1"):
        ingest.parse_permutation("0 0\n0 1\n")


def test_gtf1_corrupt_header_does_not_overflow():
    """A header whose N * f * 4 overflows (or exceeds the payload) is a
    truncation error, not a huge allocation or an out-of-bounds copy."""
    import struct

    for n, f in ((2 ** 62, 2 ** 62), (1, 2 ** 62), (2 ** 60, 1), (3, 5)):
        data = b"GTF1" + struct.pack("<QQ", n, f) + b"\0" * 16
        with pytest.raises(DataError, match="truncated at row"):
            ingest.decode_gtf1(data)
