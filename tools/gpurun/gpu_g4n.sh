# 4-GPU: NVLS reduce knob sweep at 25M (switch reductions in flight per thread, reduce CTA shape)
O=gpurun_out/${OUT:-g4n}; mkdir -p $O
i=0
for cfg in "4 120 0.5" "2 120 0.5" "8 120 0.5" "4 120 0.75" "8 120 0.75" "4 0 0.5" "8 0 1.0" "4 120 0.5"; do
  set -- $cfg; i=$((i+1))
  DSGD_NVLS_UNROLL=$1 DSGD_AR_COMM_SMEM=$2 DSGD_AR_COMM_FRAC=$3 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29670 + i)) bench.py --gpus 4 --no-extras --no-cpu > $O/bench_u$1_s$2_c$3_$i.json 2> $O/bench_$i.err
  echo run$i=$? >> $O/status.txt
done
