# 4-GPU debug: in-process p=4 crash backtrace, binding under MALLOC_PERTURB_, k_local_tma variants
O=gpurun_out/g4c; mkdir -p $O
export PYTHONFAULTHANDLER=1
for be in default p2p; do
  if [ $be = p2p ]; then export DSGD_ALLREDUCE=p2p; fi
  LD_PRELOAD=$PWD/tools/debug/segv_trace.so timeout 120 python tools/nvlink_profile.py --gpus 4 --protocol pull-gossip --rounds 5 > $O/n4_pull_$be.log 2>&1; echo n4_pull_$be=$? >> $O/status.txt
  LD_PRELOAD=$PWD/tools/debug/segv_trace.so timeout 120 python tools/nvlink_profile.py --gpus 3 --protocol pull-gossip --rounds 5 > $O/n3_pull_$be.log 2>&1; echo n3_pull_$be=$? >> $O/status.txt
done
unset DSGD_ALLREDUCE
MALLOC_PERTURB_=165 timeout 300 python -m pytest tests/test_reference_binding.py -q -x -k drivers > $O/bind_perturb.log 2>&1; echo bind_perturb=$? >> $O/status.txt
for i in 1 2; do
  timeout 120 python tools/step_gap.py > $O/gap_chain_$i.txt 2>&1
  DSGD_LT_CHAIN=0 timeout 120 python tools/step_gap.py > $O/gap_nochain_$i.txt 2>&1
  timeout 120 python ab_tmp/r1/step_gap.py > $O/gap_r1_$i.txt 2>&1
done
DSGD_PDL=0 DSGD_LT_CHAIN=0 timeout 120 python tools/step_gap.py > $O/gap_nopdl.txt 2>&1
