# 2-GPU: all-reduce tracer at 1M / 4M / 25M per worker (wait / work / launch gap per kernel)
O=gpurun_out/${OUT:-g2h}; mkdir -p $O
for d in 1000000 4000000 25000000; do
  DSGD_TRACE=4096 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 tools/trace_allreduce.py --params $d --rounds 40 > $O/trace_n2_$d.log 2>&1; echo trace_$d=$? >> $O/status.txt
done
