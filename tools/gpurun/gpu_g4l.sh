# 4-GPU: N=4 all-reduce regression bisect (PDL, gpu-scope signal)
O=gpurun_out/${OUT:-g4l}; mkdir -p $O
i=0
for cfg in "1 1" "0 1" "1 0" "0 0" "1 1"; do
  set -- $cfg; i=$((i+1))
  DSGD_PDL=$1 DSGD_SIGNAL_GPU=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29660 + i)) bench.py --gpus 4 --no-extras --no-cpu > $O/bench_pdl$1_sig$2_$i.json 2> $O/bench_$i.err
  echo run$i=$? >> $O/status.txt
done
