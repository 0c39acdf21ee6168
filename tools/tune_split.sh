# N = 4 NVLS two-shot: delta / reduce CTAs on disjoint SMs (comm smem pad, 1024-thread reduce CTAs)
mkdir -p gpurun_out/split3
i=0
for cfg in "1.5 0.5 120" "1.75 0.5 120" "2 0.5 120" "1.5 0.25 120" "1.5 0.75 120" "2 0.25 120"; do
  set -- $cfg; i=$((i+1))
  DSGD_AR_DELTA_FRAC=$1 DSGD_AR_COMM_FRAC=$2 DSGD_AR_COMM_SMEM=$3 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800+i)) tools/trace_allreduce.py > gpurun_out/split3/t_$1_$2_$3_$i.log 2>&1
done
