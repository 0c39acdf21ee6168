# 2-GPU: staged EASGD chain grid-size sweep (CTAs per SM)
O=gpurun_out/${OUT:-g2n}; mkdir -p $O
for f in 1.0 0.9 0.75 0.5 1.0; do
  DSGD_EA_GRID=$f timeout 120 python tools/nvlink_profile.py --gpus 2 --protocol elastic-avg --rounds 30 | sed "s/^{/{\"grid\": $f, /" >> $O/wall.jsonl 2>> $O/wall.err
done
