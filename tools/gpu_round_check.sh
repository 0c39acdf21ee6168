set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_gpu4.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 300 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo n1=$? >> gpurun_out/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2=$? >> gpurun_out/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo n4=$? >> gpurun_out/status.txt
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_n1.json 2>&1; echo ref=$? >> gpurun_out/status.txt
