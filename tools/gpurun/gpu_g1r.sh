# 1-GPU round check: the driver's GPU tier (pytest -m gpu, smoke), bench N=1 + reference arm,
# then the ncu launch list and one --set full capture of the dominant kernel.
O=gpurun_out/${OUT:-g1r}; mkdir -p $O/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rfs > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/status.txt
timeout 400 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo n1=$? >> $O/status.txt
timeout 400 python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err; echo ref=$? >> $O/status.txt
CMD="python bench.py --steps 20 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > $O/ncu/bench_plain.json 2> $O/ncu/bench_plain.err; echo plain=$? >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu/launches_n1.csv $CMD > $O/ncu/ncu_launch.log 2>&1; echo launches=$? >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_tma -s 5 -c 1 -o $O/ncu/prof_local_tma $CMD > $O/ncu/ncu_full.log 2>&1; echo full=$? >> $O/status.txt
