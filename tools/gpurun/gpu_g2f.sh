# 2-GPU: resident run_sync repeatability; small-d latency probe
O=gpurun_out/${OUT:-g2f}; mkdir -p $O
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_reference_binding.py -q -rf -k "resident or drivers" > $O/bind_$i.log 2>&1; echo bind_$i=$? >> $O/status.txt
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/small_d_probe.py > $O/small_d_n2.jsonl 2> $O/small_d_n2.err; echo small_d=$? >> $O/status.txt
