# 4-GPU: NVLS reduce knob sweep, round 2 (unroll 1/2, reduce CTAs per SM, pipelines)
O=gpurun_out/${OUT:-g4o}; mkdir -p $O
i=0
for cfg in "2 0.5 2" "1 0.5 2" "2 0.4 2" "2 0.6 2" "1 0.6 2" "2 0.5 4" "2 0.5 2" "1 0.5 2"; do
  set -- $cfg; i=$((i+1))
  DSGD_NVLS_UNROLL=$1 DSGD_AR_COMM_FRAC=$2 DSGD_AR_PIPES=$3 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29680 + i)) bench.py --gpus 4 --no-extras --no-cpu > $O/bench_u$1_c$2_p$3_$i.json 2> $O/bench_$i.err
  echo run$i=$? >> $O/status.txt
done
for u in 2 1; do
  DSGD_NVLS_UNROLL=$u timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29690 + u)) bench.py --gpus 4 --params 1000000000 --steps 10 --warmup 3 --no-extras --no-cpu > $O/bench_1b_u$u.json 2> $O/bench_1b_u$u.err
done
