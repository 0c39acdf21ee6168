# 2-GPU: PDL on the multi-GPU kernels -- parity, small-d latency and bench A/B
O=gpurun_out/${OUT:-g2g}; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py tests/test_inproc_ranks.py -q -rf -x > $O/pytest.log 2>&1; echo pytest=$? >> $O/status.txt
for pdl in 1 0; do
  DSGD_PDL=$pdl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29580 + pdl)) tools/small_d_probe.py --sizes 1e6,4e6,25e6 | sed "s/^{/{\"pdl\": $pdl, /" >> $O/small_d.jsonl 2>> $O/small_d.err
  DSGD_PDL=$pdl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29590 + pdl)) bench.py --gpus 2 --no-cpu > $O/bench_n2_pdl$pdl.json 2> $O/bench_n2_pdl$pdl.err
  echo pdl$pdl=$? >> $O/status.txt
done
