# 4-GPU: NVLS split fine sweep with 2 reductions in flight per thread (25M per worker)
O=gpurun_out/${OUT:-g4q}; mkdir -p $O
i=0
for cfg in "1.5 0.5" "1.5 0.47" "1.5 0.54" "1.4 0.5" "1.6 0.5" "1.3 0.5" "1.75 0.5" "1.5 0.5"; do
  set -- $cfg; i=$((i+1))
  DSGD_AR_DELTA_FRAC=$1 DSGD_AR_COMM_FRAC=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + i)) bench.py --gpus 4 --no-extras --no-cpu > $O/bench_d$1_c$2_$i.json 2> $O/bench_$i.err
  echo run$i=$? >> $O/status.txt
done
