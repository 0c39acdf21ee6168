"""Host side of the logistic objective (no GPU): the LogisticObjective
mirror's constructor checks (objectives.cpp:80-106) and load_csv_dataset
(objectives.cpp:195-248), written after test_objectives.cpp."""
import numpy as np
import pytest

from paper_1611_04581_b200 import protocols as P


def tiny(l2=0.1):
    return P.LogisticObjective([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0], [-1.0, 0.5]],
                               [1, 0, 1, 0], l2)


def test_constructor_checks():
    o = tiny()
    assert o.dim() == 2 and o.num_samples() == 4 and o.optimum() is None
    m, L = o.convexity_params()
    assert m == 0.1 and L == pytest.approx(0.1 + 0.25 * 2.0)
    with pytest.raises(P.InvalidArgument, match="empty"):
        P.LogisticObjective([], [], 0.1)
    with pytest.raises(P.InvalidArgument, match="size mismatch"):
        P.LogisticObjective([[1.0]], [0, 1], 0.1)
    with pytest.raises(P.InvalidArgument, match="positive"):
        tiny(0.0)
    with pytest.raises(P.InvalidArgument, match="inconsistent width"):
        P.LogisticObjective([[1.0], [1.0, 2.0]], [0, 1], 0.1)
    with pytest.raises(P.InvalidArgument, match="0 or 1"):
        P.LogisticObjective([[1.0], [2.0]], [0, 2], 0.1)
    with pytest.raises(P.InvalidArgument, match="invalid sample range"):
        o.set_sample_range(2, 2)
    with pytest.raises(P.InvalidArgument, match="invalid sample range"):
        o.set_sample_range(0, 5)
    s = o.shard(1, 3)
    assert s.range == (1, 3) and o.range == (0, 4)


def test_load_csv(tmp_path):
    f = tmp_path / "d.csv"
    f.write_text("label,a,b\r\n1, 0.5 ,2\r\n\r\n0,-1,3e-1\n")
    o = P.load_csv_dataset(str(f), True, 0.2)
    assert o.labels.tolist() == [1, 0]
    assert o.features.tolist() == [[0.5, 2.0], [-1.0, 0.3]]
    cases = {"1,2\n0,x\n": "line 2: field 'x' is not a number",
             "1,2\n1\n": "line 2: expected label plus at least one feature",
             "2,1\n": "line 1: label must be 0 or 1",
             "1,2\n0,1,2\n": "line 2: row width differs from first row",
             "1,2abc\n": "line 1: field '2abc' is not a number",
             "\n\n": "dataset has no rows"}
    for text, msg in cases.items():
        f.write_text(text)
        with pytest.raises(RuntimeError, match=msg):
            P.load_csv_dataset(str(f), False, 0.1)
    with pytest.raises(RuntimeError, match="cannot open dataset"):
        P.load_csv_dataset(str(tmp_path / "missing.csv"), False, 0.1)
