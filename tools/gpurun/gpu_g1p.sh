# 1-GPU: GPU tier after PDL on the staged step kernel; async-event A/B
O=gpurun_out/${OUT:-g1p}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rfs -x > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 400 python bench.py --no-cpu > $O/bench_n1.json 2> $O/bench_n1.err; echo n1=$? >> $O/status.txt
DSGD_PDL=0 timeout 400 python bench.py --no-cpu > $O/bench_n1_nopdl.json 2> $O/bench_n1_nopdl.err; echo n1_nopdl=$? >> $O/status.txt
