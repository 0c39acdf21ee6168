# bench.py at N = 1, 2, 4 on one box (outputs under gpurun_out/ba/)
mkdir -p gpurun_out/ba
timeout 300 python bench.py > gpurun_out/ba/n1.json 2> gpurun_out/ba/n1.err; echo n1=$? >> gpurun_out/ba/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29761 bench.py --gpus 2 > gpurun_out/ba/n2.json 2> gpurun_out/ba/n2.err; echo n2=$? >> gpurun_out/ba/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29762 bench.py --gpus 4 > gpurun_out/ba/n4.json 2> gpurun_out/ba/n4.err; echo n4=$? >> gpurun_out/ba/status.txt
