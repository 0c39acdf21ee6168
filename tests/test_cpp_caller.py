"""The C++ drop-in header (include/dsgd_b200.hpp) compiles and links
against libdsgd_b200.so (CPU), and a reference-style C++ caller reproduces
test_protocols.cpp hand values on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "reference_style.cpp")
LIBDIR = os.path.join(ROOT, "paper_1611_04581_b200")


def build(tmp_path):
    exe = os.path.join(str(tmp_path), "reference_style")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-ldsgd_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_header_builds_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_caller_runs_on_gpu(tmp_path):
    exe = build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "all checks passed" in out.stdout


def build_worker(tmp_path):
    exe = os.path.join(str(tmp_path), "dsgd_worker")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "cpp", "dsgd_worker.cpp"), "-L", LIBDIR,
                    "-ldsgd_b200", f"-Wl,-rpath,{LIBDIR}", "-lpthread", "-o", exe], check=True)
    return exe


def test_cpp_multiprocess_worker_builds(tmp_path):
    assert os.path.exists(build_worker(tmp_path))


@pytest.mark.gpu
def test_cpp_multiprocess_worker_runs(tmp_path):
    """C++-only host (fork per GPU, shared-memory handle exchange, NCCL id,
    dsgd_run_rounds): the run_transport counterpart without Python."""
    import json
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    exe = build_worker(tmp_path)
    for proto in ("all-reduce", "pull-gossip", "elastic-avg"):
        out = subprocess.run([exe, "--gpus", "2", "--d", "1000003", "--rounds", "20",
                              "--protocol", proto], capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stdout + out.stderr
        j = json.loads(out.stdout.strip().splitlines()[-1])
        assert j["ok"] is True and j["param_updates_per_s"] > 0


@pytest.mark.gpu
def test_cpp_worker_nvls_without_torch(tmp_path):
    """p > 2 from a C++-only host: the library creates the NVSwitch
    multicast object itself (cuMulticastCreate, pidfd_getfd, bind) and the
    all-reduce runs in the switch; every rank ends bit-identical."""
    import json
    import torch
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    exe = build_worker(tmp_path)
    out = subprocess.run([exe, "--gpus", "4", "--d", "25000000", "--rounds", "30",
                          "--protocol", "all-reduce"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    j = json.loads(out.stdout.strip().splitlines()[-1])
    assert j["ok"] is True and j["ranks_identical"] is True
    assert j["allreduce_backend"] == "nvls", j
