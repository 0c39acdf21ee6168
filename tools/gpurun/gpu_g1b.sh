# 1-GPU: chained k_local_tma rounds vs round-1 library (same box), parity, bench
O=gpurun_out/g1b; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fp32_tolerance.py -q -x -k "allreduce or local" > $O/pytest_ar.log 2>&1; echo pytest_ar=$? >> $O/status.txt
for i in 1 2; do
  timeout 120 python tools/step_gap.py > $O/gap_new_$i.txt 2>&1
  timeout 120 python ab_tmp/r1/step_gap.py > $O/gap_r1_$i.txt 2>&1
done
DSGD_PDL=0 timeout 120 python tools/step_gap.py > $O/gap_new_nopdl.txt 2>&1
timeout 400 python bench.py --no-cpu > $O/bench_n1.json 2> $O/bench_n1.err; echo n1=$? >> $O/status.txt
