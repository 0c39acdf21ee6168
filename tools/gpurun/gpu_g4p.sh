# 4-GPU final bench lines (N=2, N=4 with extras) and the reference arm at N=4
O=gpurun_out/${OUT:-g4p}; mkdir -p $O
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2=$? >> $O/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo n4=$? >> $O/status.txt
timeout 300 python bench.py --impl reference --gpus 4 > $O/bench_ref_n4.json 2> $O/bench_ref_n4.err; echo ref4=$? >> $O/status.txt
timeout 300 python bench.py --impl reference --gpus 2 > $O/bench_ref_n2.json 2> $O/bench_ref_n2.err; echo ref2=$? >> $O/status.txt
