# 2-GPU: small-d fixed cost -- N=1 bench at 1M/4M, N=2 one-shot CTA-count variants
O=gpurun_out/${OUT:-g2i}; mkdir -p $O
for d in 1000000 4000000; do
  timeout 300 python bench.py --params $d --no-extras --no-cpu --steps 200 > $O/bench_n1_$d.json 2> $O/bench_n1_$d.err
done
for c in 1 2 0; do
  DSGD_OS_CTAS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29610 + c)) tools/small_d_probe.py --sizes 1e6,4e6 --protocols all-reduce | sed "s/^{/{\"os_ctas\": $c, /" >> $O/ctas.jsonl 2>> $O/ctas.err
done
