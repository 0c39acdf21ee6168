# 2-GPU: per-round latency floor (tiny d) for every multi-GPU protocol
O=gpurun_out/${OUT:-g2j}; mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/small_d_probe.py --sizes 4096,65536,1e6 > $O/tiny.jsonl 2> $O/tiny.err; echo tiny=$? >> $O/status.txt
for d in 4096 65536; do
  DSGD_TRACE=4096 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 tools/trace_allreduce.py --params $d --rounds 40 > $O/trace_$d.log 2>&1
done
