# 4-GPU final parity subset: NVLS (2 reductions in flight), two-shot pipelines, default protocols, C++ NVLS worker
O=gpurun_out/${OUT:-g4r}; mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_cpp_caller.py -q -rA --timeout 900 -k "nvls or two_shot or default or missing_peer or three_ranks" > $O/pytest.log 2>&1; echo pytest=$? >> $O/status.txt
