# 4-GPU: hunt the resident run_sync flake (repeat, then after in-process groups, then the g4h order)
O=gpurun_out/${OUT:-g4i}; mkdir -p $O
REPS=10 timeout 600 python tools/debug/resident_repro.py > $O/repro_plain.log 2>&1; echo plain=$? >> $O/status.txt
REPS=10 timeout 900 python tools/debug/resident_repro.py inproc > $O/repro_inproc.log 2>&1; echo inproc=$? >> $O/status.txt
timeout 1200 python -m pytest tests/test_inproc_ranks.py tests/test_reference_binding.py -q -rf > $O/pytest_order.log 2>&1; echo order=$? >> $O/status.txt
