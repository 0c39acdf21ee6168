# 4-GPU final-code check: the multi-GPU suite, bench N=2/4, gossip / EASGD tracer at N=4
O=gpurun_out/${OUT:-g4k}; mkdir -p $O
timeout 1800 python -m pytest tests/test_multigpu.py tests/test_inproc_ranks.py tests/test_reference_binding.py tests/test_cpp_caller.py -q -rA --timeout 900 > $O/pytest_mgpu.log 2>&1; echo pytest_mgpu=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$? >> $O/status.txt
for p in pull-gossip elastic-avg all-reduce; do
  d=25000000; [ $p = pull-gossip ] && d=10000000
  DSGD_TRACE=4096 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 tools/trace_allreduce.py --protocol $p --params $d --rounds 40 > $O/trace_n4_$p.log 2>&1; echo trace_$p=$? >> $O/status.txt
done
