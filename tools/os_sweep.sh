# one-shot all-reduce (N = 2) staging sweep: stages x CTAs per SM
mkdir -p gpurun_out/os2
i=0
for cfg in "2 0" "3 0" "2 1" "2 3" "2 0" "3 0"; do
  set -- $cfg; i=$((i+1))
  DSGD_OS_STAGES=$1 DSGD_OS_CTAS=$2 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29680+i)) bench.py --gpus 2 --no-extras --steps 50 > gpurun_out/os2/bench_s$1_c$2_$i.json 2> gpurun_out/os2/bench_s$1_c$2_$i.err
done
