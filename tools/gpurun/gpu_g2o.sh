# 2-GPU: ncu --set full of the multi-GPU kernels (in-process group, one launch each)
O=gpurun_out/${OUT:-g2o}; mkdir -p $O
for p in elastic-avg all-reduce pull-gossip; do
  timeout 120 python tools/nvlink_profile.py --gpus 2 --protocol $p --rounds 2 --warmup 1 > $O/plain_$p.log 2>&1 || continue
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ea_chain_tma -s 2 -c 1 -o $O/prof_ea_chain python tools/nvlink_profile.py --gpus 2 --protocol elastic-avg --rounds 2 --warmup 1 > $O/ncu_ea.log 2>&1; echo ea=$? >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ar_oneshot_tma2 -s 2 -c 1 -o $O/prof_oneshot python tools/nvlink_profile.py --gpus 2 --protocol all-reduce --rounds 2 --warmup 1 > $O/ncu_os.log 2>&1; echo os=$? >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_step_tma2<float, 1>" -s 1 -c 1 -o $O/prof_pull python tools/nvlink_profile.py --gpus 2 --protocol pull-gossip --rounds 2 --warmup 1 > $O/ncu_pull.log 2>&1; echo pull=$? >> $O/status.txt
