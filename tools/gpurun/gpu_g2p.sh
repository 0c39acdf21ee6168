# 2-GPU: one-shot all-reduce staging re-check (stages x CTAs per SM) with the round-2 launch/signal path
O=gpurun_out/${OUT:-g2p}; mkdir -p $O
i=0
for cfg in "2 0" "3 0" "2 2" "4 0" "2 0"; do
  set -- $cfg; i=$((i+1))
  DSGD_OS_STAGES=$1 DSGD_OS_CTAS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29720 + i)) bench.py --gpus 2 --no-extras --no-cpu > $O/bench_s$1_c$2_$i.json 2> $O/bench_$i.err
done
