# 2-GPU: EASGD chain with 1024-element chunks and two CTAs per SM (DSGD_EA_TILE_U=1) -- parity + A/B
O=gpurun_out/${OUT:-g2r}; mkdir -p $O
DSGD_EA_TILE_U=1 timeout 600 python -m pytest tests/test_inproc_ranks.py tests/test_multigpu.py -q -rf -x -k "elastic or (protocols and default and f32) or missing_peer" > $O/pytest_u1.log 2>&1; echo pytest_u1=$? >> $O/status.txt
for u in 2 1 2 1; do
  DSGD_EA_TILE_U=$u timeout 120 python tools/nvlink_profile.py --gpus 2 --protocol elastic-avg --rounds 30 | sed "s/^{/{\"u\": $u, /" >> $O/wall.jsonl 2>> $O/wall.err
done
for u in 2 1; do
  DSGD_EA_TILE_U=$u timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29760 + u)) bench.py --gpus 2 --no-cpu > $O/bench_n2_u$u.json 2> $O/bench_n2_u$u.err
done
