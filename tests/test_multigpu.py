"""Multi-GPU parity (>= 2 GPUs): one process per GPU under torchrun.  The
NVLink peer-read gossip kernels, the EASGD chain and the peer-memory
all-reduce (reference ring order) must match the oracle bit-for-bit (the
all-reduce: the reference's threaded transport, run_transport); the NCCL
all-reduce backend within 1e-12 / 1e-5 (NCCL's summation order is its own)
with every rank bit-identical."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def n_gpus():
    import torch
    return torch.cuda.device_count()


BACKENDS = ["default", "oneshot", "p2p", "nvls", "nccl"]


def worlds():
    try:
        n = n_gpus()
    except Exception:
        n = 0
    return [w for w in (2, 4, 8) if w <= n] or [2]


@pytest.mark.skipif("n_gpus() < 2")
@pytest.mark.parametrize("world", worlds())
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("backend", BACKENDS)
def test_multi_gpu_protocols_match_oracle(world, dtype, backend):
    if backend == "oneshot" and world > 4:
        pytest.skip("one-shot all-reduce is for p <= 4")
    port = 29611 + 16 * (world // 2) + (dtype == "f32") + 2 * BACKENDS.index(backend)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mgpu_worker.py"), dtype]
    env = dict(os.environ)
    if backend != "default":   # default at p = 2: the one-shot peer-memory kernel
        cmd.append("allreduce-only")
        env["DSGD_ALLREDUCE"] = backend
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT ")][0]
    res = json.loads(line[7:])
    for proto, r in res.items():
        assert r["ranks_identical"] or proto != "all-reduce", proto
        if proto.startswith("all-reduce") and (backend == "nccl" or r["nvls"]):
            assert r["max_rel"] <= (1e-12 if dtype == "f64" else 1e-5), (proto, r)
        else:
            assert r["bit_exact"], (proto, r)
        if r["center_exact"] is not None:
            assert r["center_exact"], (proto, r)


@pytest.mark.skipif("n_gpus() < 2")
@pytest.mark.parametrize("world", worlds())
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_multi_gpu_logistic_matches_single_context(world, dtype):
    """F1 across GPUs: the device logistic gradient with sharded sample
    ranges, one node per GPU, against the single-context run (gossip/EASGD
    bit-exact; all-reduce within 1e-12 / 1e-5: ring vs pivot summation)."""
    port = 29711 + 4 * (world // 2) + (dtype == "f32")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mgpu_worker.py"), dtype, "logistic"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT ")][0]
    res = json.loads(line[7:])
    assert set(res) == {"all-reduce", "elastic-avg", "pull-gossip", "push-gossip",
                        "gossip-stale", "gossip-fresh"}
    for proto, r in res.items():
        assert r["t_ok"], (proto, r)
        if proto == "all-reduce":
            assert r["max_rel"] <= (1e-12 if dtype == "f64" else 1e-5), (proto, r)
        else:
            assert r["bit_exact"], (proto, r)
        if "center_exact" in r:
            assert r["center_exact"], (proto, r)


@pytest.mark.skipif("n_gpus() < 2")
def test_multi_gpu_missing_peer_times_out():
    """A peer that never runs its round: the waiting kernel gives up after
    the context timeout (%globaltimer-bounded flag waits) and the call
    surfaces TransportError -- for the gossip RAW wait, the all-reduce and
    the EASGD chain's ring closure (staged kernel: the producer warp gives up,
    every warp still finishes)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29731",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), "f32", "timeout"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT ")][0]
    res = json.loads(line[7:])
    for proto in ("pull-gossip", "all-reduce", "elastic-avg"):
        assert res[proto]["timed_out"], res
        assert "timed out" in res[proto]["message"]
        assert res[proto]["seconds"] < 20.0, res


@pytest.mark.skipif("n_gpus() < 3")
def test_multi_gpu_three_ranks_match_oracle():
    """p = 3 (uneven reference ring chunks, odd slice split): every protocol
    with the default backends against the oracle, fp64."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=3",
           "--master-addr", "127.0.0.1", "--master-port", "29741",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), "f64"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT ")][0]
    res = json.loads(line[7:])
    for proto, r in res.items():
        if proto.startswith("all-reduce") and r["nvls"]:
            assert r["max_rel"] <= 1e-12, (proto, r)
        else:
            assert r["bit_exact"], (proto, r)
        if r["center_exact"] is not None:
            assert r["center_exact"], (proto, r)


@pytest.mark.skipif("n_gpus() < 2")
@pytest.mark.parametrize("backend,pipes", [("nvls", 4), ("nvls", 2), ("p2p", 4)])
def test_multi_gpu_two_shot_pipelines(backend, pipes):
    """The two-shot all-reduce at a size that splits d into pipelines
    (8M + 1031 per rank, both momentum scopes): the NVLS reduce on its own
    SMs with 2 / 4 pipelines (the >= 700M default) within tolerance and
    every rank identical; the peer-memory ring reduce bit-exact with the
    reference's threaded transport."""
    world = min(4, n_gpus())
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(29751 + pipes + (backend == "p2p")),
           os.path.join(ROOT, "tests", "mgpu_worker.py"), "f32", "allreduce-only"]
    env = dict(os.environ, DSGD_ALLREDUCE=backend, DSGD_AR_PIPES=str(pipes),
               MGPU_AR_D=str((8 << 20) + 1031), MGPU_ROUNDS="6")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    res = json.loads([l for l in out.stdout.splitlines() if l.startswith("RESULT ")][0][7:])
    for proto, r in res.items():
        assert r["ranks_identical"], (proto, r)
        if r["nvls"]:
            assert r["max_rel"] <= 1e-5, (proto, r)
        else:
            assert r["bit_exact"], (proto, r)
