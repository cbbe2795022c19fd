"""Trainer glue: pad loops, SPD bias buckets, bias gather
and table gradient. Golden: tests/golden/glue_small.npz (the compiled
reference's spd_table, layouts, and the bucket fill restated in the C oracle,
tests/golden/make_glue_golden.py)."""
import numpy as np
import pytest

from oracle import CSR

from paper_2407_14106_b200 import glue

CASES = (0, 1, 2)


def _case(golden, ci):
    d = golden("glue_small.npz")
    return {k[len(f"c{ci}_"):]: d[k] for k in d.files if k.startswith(f"c{ci}_")}


def _py_buckets(c):
    """Direct restatement of model.cpp:447-463 + SpdTable::lookup in numpy."""
    ro, co, inv = c["pat_ro"], c["pat_cols"], c["inv_pad"]
    sro, scol, sdist, sn = c["spd_ro"], c["spd_cols"], c["spd_dist"], int(c["spd_n"])
    un, glob = int(c["cap"]) + 1, int(c["glob"])
    out = []
    for r in range(ro.shape[0] - 1):
        for cc in co[ro[r]:ro[r + 1]]:
            i, j = inv[r], inv[cc]
            if i == j:
                out.append(0)
            elif i == glob or j == glob:
                out.append(1)
            elif i >= sn or j >= sn:
                out.append(un)
            else:
                row = scol[sro[i]:sro[i + 1]]
                p = np.searchsorted(row, j)
                out.append(int(sdist[sro[i] + p]) if p < row.shape[0] and row[p] == j else un)
    return np.array(out, dtype=np.int32)


@pytest.mark.parametrize("ci", CASES)
def test_oracle_buckets_golden(orc, golden, ci):
    c = _case(golden, ci)
    pat = CSR(int(c["pat_ro"].shape[0] - 1), c["pat_ro"], c["pat_cols"])
    spd = (c["spd_ro"], c["spd_cols"], c["spd_dist"], int(c["spd_n"]))
    got = orc.pattern_buckets(pat, c["inv_pad"], int(c["glob"]), spd, int(c["cap"]))
    assert np.array_equal(got, c["buckets"])
    assert np.array_equal(_py_buckets(c), c["buckets"])


@pytest.mark.parametrize("ci", CASES)
def test_extend_with_pad_loops(orc, golden, ci):
    c = _case(golden, ci)
    ro, co = glue.extend_with_pad_loops(c["layout_ro"], c["layout_cols"], int(c["s_pad"]))
    assert np.array_equal(ro, c["pat_ro"]) and np.array_equal(co, c["pat_cols"])
    want = orc.extend_with_pad_loops(CSR(int(c["layout_ro"].shape[0] - 1), c["layout_ro"], c["layout_cols"]),
                                     int(c["s_pad"]))
    assert np.array_equal(want.row_off, ro) and np.array_equal(want.cols, co)


@pytest.mark.gpu
@pytest.mark.parametrize("ci", CASES)
def test_device_buckets_and_table(cuda, golden, ci):
    import torch

    c = _case(golden, ci)
    spd = (c["spd_ro"], c["spd_cols"], c["spd_dist"], int(c["spd_n"]))
    b = glue.pattern_buckets(c["pat_ro"], c["pat_cols"], c["inv_pad"], int(c["glob"]), spd, int(c["cap"]))
    assert np.array_equal(b.cpu().numpy(), c["buckets"])
    nb = int(c["cap"]) + 2
    rng = np.random.default_rng(ci)
    table = torch.tensor(rng.normal(0, 0.3, nb), dtype=torch.float32, device="cuda")
    bias = glue.bias_from_table(b, table)
    assert np.array_equal(bias.cpu().numpy(), table.cpu().numpy()[c["buckets"]])
    db = torch.tensor(rng.standard_normal(b.numel()), dtype=torch.float32, device="cuda")
    g1 = glue.dbias_to_table(b, db, nb)
    g2 = glue.dbias_to_table(b, db, nb)
    want = np.bincount(c["buckets"], weights=db.double().cpu().numpy(), minlength=nb)
    assert np.array_equal(g1.cpu().numpy(), g2.cpu().numpy())  # fixed summation order
    assert np.abs(g1.double().cpu().numpy() - want).max() <= 1e-5 * max(1.0, np.abs(want).max())
