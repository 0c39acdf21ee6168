# N = 1 profiling pass (one GPU): the bench command clean, then its ncu
# launch list, then one --set full capture of the dominant kernel.
mkdir -p gpurun_out/ncu
CMD="python bench.py --steps 20 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > gpurun_out/ncu/bench_plain.json 2> gpurun_out/ncu/bench_plain.err; echo plain=$? >> gpurun_out/ncu/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches_n1.csv $CMD > gpurun_out/ncu/ncu_launch.log 2>&1; echo launches=$? >> gpurun_out/ncu/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_tma -s 5 -c 1 -o gpurun_out/ncu/prof_local_tma $CMD > gpurun_out/ncu/ncu_full.log 2>&1; echo full=$? >> gpurun_out/ncu/status.txt
