# 4-GPU: two-shot pipeline parity at 8M, final-code bench N=2/4 and the 1B-per-worker N=4 round
O=gpurun_out/${OUT:-g4j}; mkdir -p $O
timeout 1500 python -m pytest tests/test_multigpu.py -q -rA -k "two_shot_pipelines" > $O/pytest_pipes.log 2>&1; echo pipes=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$? >> $O/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29557 bench.py --gpus 4 --params 1000000000 --steps 10 --warmup 3 --no-extras --no-cpu > $O/bench_n4_1b.json 2> $O/bench_n4_1b.err; echo n4_1b=$? >> $O/status.txt
