"""Host side of the logistic objective (no GPU): the LogisticObjective
mirror's constructor checks (objectives.cpp:80-106), written after
test_objectives.cpp."""
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
