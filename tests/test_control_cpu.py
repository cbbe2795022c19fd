"""Host control logic through the product library (csrc/host_api.cpp via
control.py) against the compiled reference's golden trajectories
(tests/golden/reformation_small.npz, tests/golden/make_golden.py): the ECR
tuner (reformation.cpp:224-265), select_k / select_db (:267-296), select_mode
(interleave.cpp:101-106). No GPU."""
import numpy as np

from paper_2407_14106_b200 import control


def test_tuner_trajectories_golden(golden):
    d = golden("reformation_small.npz")
    for ci in range(8):
        p = f"t{ci}_"
        losses, times = d[p + "in"]
        t = control.Tuner(float(d[p + "bg"]), int(d[p + "delta"]))
        idx, avg = [], []
        for e, (l, s) in enumerate(zip(losses, times)):
            t.update(float(l), float(s), e)
            a, i, thr, _ = t.state()
            idx.append(i)
            avg.append(a)
        assert np.array_equal(np.array(idx), d[p + "idx"]), ci
        assert np.array_equal(np.array(avg), d[p + "avg"]), ci
        assert np.array_equal(thr, d[p + "thr"]), ci


def test_selectors_golden(golden):
    d = golden("reformation_small.npz")
    for l2, dd, i, want in d["select_k"]:
        assert control.select_k(int(l2), int(dd), int(i)) == int(want)
    assert control.select_db([2, 8, 16, 32, 128], [1.0, 2.0, 2.4, 2.1, 1.2]) == int(d["select_db"][0]) == 16
    assert control.select_db([16], [1.0]) == int(d["select_db"][1])


def test_select_mode_rules():
    # interleave.cpp:101-106: dense on the period, dense when a condition fails, else sparse
    assert control.select_mode([1, 1, 1], 4, 4) == (1, 1)
    assert control.select_mode([1, 0, 1], 3, 4) == (1, 0)
    assert control.select_mode([1, 1, 1], 3, 4) == (0, 2)
