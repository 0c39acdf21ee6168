# 2-GPU: staged step kernel depth (DSGD_STEP_STAGES 2/3/4): N=2 gossip + 1-GPU 8-node pull / async events
O=gpurun_out/${OUT:-g2q}; mkdir -p $O
for st in 3 4 2 3; do
  DSGD_STEP_STAGES=$st timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29740 + st)) bench.py --gpus 2 --no-cpu > $O/bench_n2_st$st.json 2> $O/bench_n2_st$st.err
  DSGD_STEP_STAGES=$st timeout 300 python bench.py --no-cpu > $O/bench_n1_st$st.json 2> $O/bench_n1_st$st.err
done
