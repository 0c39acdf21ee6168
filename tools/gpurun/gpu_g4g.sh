# 4-GPU: NVLS split sweep per d (all-reduce), then the configs[4] sweep at N=2 and N=4
O=gpurun_out/${OUT:-g4g}; mkdir -p $O
i=0
for cfg in "1.5 0.5 120 2" "2 2 0 2" "1 1 120 2" "1.25 0.75 120 2" "1.5 0.5 120 4" "2 2 0 4"; do
  set -- $cfg
  i=$((i+1))
  DSGD_AR_DELTA_FRAC=$1 DSGD_AR_COMM_FRAC=$2 DSGD_AR_COMM_SMEM=$3 DSGD_AR_PIPES=$4 timeout 600 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29760 + i)) \
    tools/sweep_d.py --sizes 25e6,100e6,400e6,1e9 --protocols all-reduce --rounds 10 2>> $O/split.err | sed "s/^{/{\"split\": \"$1 $2 $3 $4\", /" >> $O/split.jsonl
  echo split$i=$? >> $O/status.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 tools/sweep_d.py > $O/sweep_n2.jsonl 2> $O/sweep_n2.err; echo sweep_n2=$? >> $O/status.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29752 tools/sweep_d.py > $O/sweep_n4.jsonl 2> $O/sweep_n4.err; echo sweep_n4=$? >> $O/status.txt
