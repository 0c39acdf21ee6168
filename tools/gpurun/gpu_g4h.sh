# 4-GPU verification: multi-GPU tests (names listed), bench N=2/4, 1B-per-worker N=4 round,
# the C++-only host (NVLS from the library, no PyTorch) at N=4
O=gpurun_out/${OUT:-g4h}; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1800 python -m pytest tests/test_multigpu.py tests/test_inproc_ranks.py tests/test_reference_binding.py tests/test_cpp_caller.py -q -rA --timeout 900 > $O/pytest_mgpu.log 2>&1; echo pytest_mgpu=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$? >> $O/status.txt
timeout 300 python bench.py --impl reference --gpus 4 > $O/bench_ref_n4.json 2> $O/bench_ref_n4.err; echo ref_n4=$? >> $O/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29557 bench.py --gpus 4 --params 1000000000 --steps 10 --warmup 3 --no-extras --no-cpu > $O/bench_n4_1b.json 2> $O/bench_n4_1b.err; echo n4_1b=$? >> $O/status.txt
for p in all-reduce elastic-avg pull-gossip; do
  timeout 300 tools/cpp/dsgd_worker --gpus 4 --d 25000000 --rounds 50 --protocol $p >> $O/cpp_worker_n4.jsonl 2>> $O/cpp_worker_n4.err; echo cpp_$p=$? >> $O/status.txt
done
