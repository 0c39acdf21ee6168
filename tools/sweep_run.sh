# configs[4] sweep at N = 2 and N = 4 (one worker per GPU)
mkdir -p gpurun_out/sweep
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 tools/sweep_d.py > gpurun_out/sweep/n2.log 2>&1; echo n2=$? >> gpurun_out/sweep/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29752 tools/sweep_d.py > gpurun_out/sweep/n4.log 2>&1; echo n4=$? >> gpurun_out/sweep/status.txt
