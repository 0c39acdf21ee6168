# N = 4 NVLS two-shot: delta / reduce CTAs on disjoint SMs (comm smem pad, 1024-thread reduce CTAs)
mkdir -p gpurun_out/split4
i=0
for cfg in "1.5 0.5 120" "1.5 0.5 100" "1.5 0.4 120" "1.4 0.6 120" "1.6 0.5 120"; do
  set -- $cfg; i=$((i+1))
  DSGD_AR_DELTA_FRAC=$1 DSGD_AR_COMM_FRAC=$2 DSGD_AR_COMM_SMEM=$3 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29830+i)) tools/trace_allreduce.py > gpurun_out/split4/t_$1_$2_$3_$i.log 2>&1
done
