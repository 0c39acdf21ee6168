# 2-GPU: gpu-scope CTA arrival for local-write kernels -- parity and latency A/B
O=gpurun_out/${OUT:-g2k}; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py -q -rf -x -k "not two_shot" > $O/pytest.log 2>&1; echo pytest=$? >> $O/status.txt
for sg in 1 0; do
  DSGD_SIGNAL_GPU=$sg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29630 + sg)) tools/small_d_probe.py --sizes 4096,1e6,25e6 | sed "s/^{/{\"sig_gpu\": $sg, /" >> $O/probe.jsonl 2>> $O/probe.err
done
