"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/dsgd_b200.h declares, its host-side pieces (streams,
schedule, step sizes, validation) match the oracle/reference, and device
calls fail loudly (status codes, no crash) when no GPU is present."""
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_1611_04581_b200 import _native as N
from paper_1611_04581_b200.engine import (Group, Hyperparams, Stream, derive_stream_seed,
                                          draw_pull_partners, draw_push_targets, step_size_at)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dsgd_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsgd_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = declared_functions()
    assert len(names) > 40
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTED), set(names) ^ set(N.EXPORTED)


def test_binary_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.SO],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_stream_seed_and_samplers_match_oracle():
    for node in (0, 3, 0xFFFFFFFF):
        for purpose in N.PURPOSE:
            assert derive_stream_seed(7, "x/trial1", node, purpose) == \
                O.derive_stream_seed(7, "x/trial1", node, purpose)
    a, b = Stream(12345), O.Stream(12345)
    assert [a.next_u64() for _ in range(700)] == [b.next_u64() for _ in range(700)]
    assert np.array([a.normal() for _ in range(100)]).tobytes() == \
        np.array([b.normal() for _ in range(100)]).tobytes()
    assert [a.uniform_index(7) for _ in range(100)] == [b.uniform_index(7) for _ in range(100)]
    assert a.exponential(2.5) == b.exponential(2.5)
    c = a.clone()
    assert a.fill_normal(0.3, 50).tobytes() == c.fill_normal(0.3, 50).tobytes()
    with pytest.raises(N.InvalidArgument):
        a.uniform_index(0)


def test_partner_draws_match_survey_kat():
    streams = [Stream.make(1, "run/trial0", i, "partner-choice") for i in range(8)]
    assert draw_pull_partners(streams).tolist() == [1, 2, 4, 3, 4, 1, 2, 7]
    assert draw_pull_partners(streams).tolist() == [0, 6, 6, 0, 0, 7, 6, 4]
    ps = [Stream.make(3, "push", i, "partner-choice") for i in range(5)]
    os_ = [O.Stream.make(3, "push", i, "partner-choice") for i in range(5)]
    for _ in range(20):
        t = draw_push_targets(ps)
        ref = []
        for i, s in enumerate(os_):
            j = s.uniform_index(4)
            ref.append(j + 1 if j >= i else j)
        assert t.tolist() == ref
        assert all(t[i] != i for i in range(5))


def test_step_size_and_validate():
    h = Hyperparams()
    assert step_size_at(h, 0) == 0.1
    assert step_size_at(h, 150000) == O.step_size_at(O.HyperParams(), 150000)
    h.validate()
    for bad in (dict(alpha0=0.0), dict(mu=1.0), dict(beta_ea=0.0), dict(tau=0),
                dict(anneal_at=(5, 3)), dict(beta_gossip=1.0)):
        hb = Hyperparams(**bad)
        with pytest.raises(N.InvalidArgument):
            hb.validate()


def test_context_errors_are_status_codes():
    with pytest.raises(N.InvalidArgument):
        Group(0, 1)
    with pytest.raises(N.InvalidArgument):
        Group(10, p=4, n_local=2)   # all p nodes or exactly one per context
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        with pytest.raises(N.DsgdError):
            Group(10, 1)   # no device: DSGD_ECUDA, not a crash
