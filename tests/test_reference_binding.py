"""The drop-in with the reference's own C++ signatures.

integration/_build/libdsgd_reference_b200.so is the reference's hot-path
library built from its UNMODIFIED sources (rng, param_vec, core, objectives,
simulator, transport) with src/protocols.cpp replaced by
integration/protocols_b200.cpp: every dsgd:: update rule of
protocols.hpp:45-152, same signatures, running on the GPU through
libdsgd_b200.so.  The reference's own run_sync / run_async / run_transport
(simulator.cpp:214-449, transport.cpp:306-553) drive it unchanged.

GPU bar: those trajectories are byte-identical (fp64) to the committed
fixtures the UNMODIFIED reference produced (tests/golden/*.npz) -- every
protocol incl. the C1 configuration's 2000 all-reduce rounds, the Poisson
drivers, the sharded LogisticObjective runs (host Objective plugin: the
gradient evaluated on the host at the rule's evaluation point) and the
threaded transport (p worker threads, each with its own device context).
"""
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "integration", "_build")
LIB = os.path.join(BUILD, "libdsgd_reference_b200.so")
HARNESS = os.path.join(BUILD, "libdsgd_ref_b200_harness.so")
GOLD = os.path.join(ROOT, "tests", "golden")

RULES = ["local_sgd_step", "compute_local_delta", "allreduce_round", "ea_client_step",
         "ea_server_apply", "pull_mix", "pull_gossip_round", "push_mix", "push_gossip_round",
         "gossip_stale_step", "gossip_fresh_step", "gossip_fresh_mix", "async_pull_event"]

needs_lib = pytest.mark.skipif(not os.path.exists(HARNESS),
                               reason="integration/_build not built (needs /root/reference)")


@needs_lib
def test_binding_exports_reference_signatures_over_the_c_abi():
    """Every protocols.hpp function is defined in the drop-in library with
    the reference's mangled signature, and the library calls the C ABI (the
    rules are not the reference's CPU code)."""
    defined = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True,
                             text=True, check=True).stdout
    for r in RULES:
        assert f" dsgd::{r}(" in defined, r
    for overload in ("dsgd::allreduce_round(std::vector<dsgd::NodeState",
                     "dsgd::run_sync(dsgd::SimConfig const&, dsgd::Objective const&)",
                     "dsgd::run_transport("):
        assert overload in defined, overload
    undefined = subprocess.run(["nm", "-D", "--undefined-only", LIB], capture_output=True,
                               text=True, check=True).stdout
    for sym in ("dsgd_allreduce_round", "dsgd_pull_gossip_round", "dsgd_push_gossip_round",
                "dsgd_ea_client_event", "dsgd_ea_server_apply", "dsgd_gossip_stale_step",
                "dsgd_mix_toward", "dsgd_async_pull_event", "dsgd_local_sgd_step"):
        assert sym in undefined, sym


def same(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


def run_cases():
    from tests.golden.make_golden import RUN_CASES
    return RUN_CASES


@pytest.mark.gpu
@needs_lib
@pytest.mark.parametrize("name", sorted(run_cases()))
def test_reference_drivers_through_binding_match_golden(name):
    """The reference's run_sync / run_async (unmodified simulator.cpp) with
    the B200 rules: byte-identical to the reference's own output."""
    cfg = run_cases()[name]
    g = np.load(os.path.join(GOLD, "runs.npz"))
    with O.ref_library(HARNESS):
        O.ref_set_logistic(None, None, 0.0)
        th, dp, t, c = O.ref_run(cfg)
    assert same(th, g[f"{name}_theta"])
    assert same(dp, g[f"{name}_dprev"])
    assert t.tolist() == g[f"{name}_t"].tolist()
    if cfg.protocol == O.ELASTIC:
        assert same(c, g[f"{name}_center"])


@pytest.mark.gpu
@needs_lib
@pytest.mark.parametrize("name", ["lg_allreduce", "lg_allreduce_agg", "lg_pull", "lg_push",
                                  "lg_ea", "lg_stale", "lg_fresh", "lg_async", "lg_ea_poisson"])
def test_logistic_objective_plugin_through_binding_matches_golden(name):
    """A host Objective (LogisticObjective, sharded sample ranges): the
    binding calls stochastic_gradient at the rule's evaluation point exactly
    as protocols.cpp does; the device applies weight decay, noise, momentum,
    mix and update in the reference order -> byte-identical trajectories."""
    from tests.golden.make_golden import LOGISTIC_CASES
    gold = np.load(os.path.join(GOLD, "logistic.npz"))
    with O.ref_library(HARNESS):
        O.ref_set_logistic(gold["X"], gold["y"], float(gold["l2"]), gold["ranges"])
        try:
            th, dp, t, c = O.ref_run(LOGISTIC_CASES[name])
        finally:
            O.ref_set_logistic(None, None, 0.0)
    assert same(th, gold[f"{name}_theta"])
    assert same(dp, gold[f"{name}_dprev"])
    assert t.tolist() == gold[f"{name}_t"].tolist()


@pytest.mark.gpu
@needs_lib
@pytest.mark.parametrize("p", [2, 4, 8])
def test_threaded_transport_through_binding_matches_golden(p):
    """run_transport (transport.cpp:306-553): p worker threads, each calling
    compute_local_delta on its own device context, the reference's mailbox
    ring all-reduce in between -> the reference's own fixture."""
    from tests.golden.make_golden import transport_case
    gold = np.load(os.path.join(GOLD, "transport.npz"))
    with O.ref_library(HARNESS):
        th, dp, t, _ = O.ref_run(transport_case(p), transport=True, chaos_seed=p)
    assert same(th, gold[f"p{p}_theta"])
    assert same(dp, gold[f"p{p}_dprev"])


@pytest.mark.gpu
@needs_lib
def test_binding_errors_keep_reference_types():
    """protocols.cpp's std::invalid_argument cases surface unchanged
    (ref_round's error path returns the exception text)."""
    h = O.HyperParams(alpha0=0.1, anneal_at=())
    with O.ref_library(HARNESS):
        n = O.Nodes(np.ones((2, 3)), t=np.array([0, 1], dtype=np.uint64))
        with pytest.raises(ValueError, match="synchronous round requires equal node clocks"):
            O.ref_round("allreduce", n, h, spec=np.ones(3))
        n = O.Nodes(np.ones((2, 3)))
        with pytest.raises(ValueError, match="partner index out of range"):
            O.ref_round("pull", n, h, partner=np.array([0, 5], dtype=np.uint32), spec=np.ones(3))
        with pytest.raises(ValueError, match="push target must differ from sender"):
            O.ref_round("push", n, h, partner=np.array([0, 0], dtype=np.uint32), spec=np.ones(3))


@pytest.mark.gpu
@needs_lib
@pytest.mark.parametrize("name", sorted(n for n, c in run_cases().items()
                                        if not c.poisson and c.protocol != O.ASYNC_PULL))
def test_resident_run_sync_matches_golden(name):
    """integration/run_sync_b200.cpp: run_sync with
    the node state on the GPU for the whole run (one dsgd_run_rounds) --
    byte-identical final state, and max_grad_norm (accumulated on the
    device, read once) equal to the reference's within its summation order."""
    cfg = run_cases()[name]
    g = np.load(os.path.join(GOLD, "runs.npz"))
    with O.ref_library(HARNESS):
        th, dp, t, c, gn = O.ref_run_resident(cfg)
    assert same(th, g[f"{name}_theta"])
    assert same(dp, g[f"{name}_dprev"])
    assert t.tolist() == g[f"{name}_t"].tolist()
    if cfg.protocol == O.ELASTIC:
        assert same(c, g[f"{name}_center"])
    if O.ref_available():  # this container: the unmodified reference's own number
        assert gn == pytest.approx(O.ref_run_max_grad_norm(cfg), rel=1e-12)
    assert gn > 0.0
