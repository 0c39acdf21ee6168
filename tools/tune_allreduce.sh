mkdir -p gpurun_out/tune2
i=0
for cfg in "2 0.25 2" "2 0.5 2" "2 0.5 1" "2 1 1" "2 0.25 1" "3 0.5 2" "4 0.5 2" "4 0.25 2" "2 2 2"; do
  set -- $cfg
  i=$((i+1))
  DSGD_AR_PIPES=$1 DSGD_AR_DELTA_FRAC=$2 DSGD_AR_COMM_FRAC=$3 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600+i)) tools/trace_allreduce.py > gpurun_out/tune2/tune_nvls_$1_$2_$3.log 2>&1
done
