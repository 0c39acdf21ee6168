# 1-GPU: k_local_tma variants (chain / no chain / no PDL / round-1 library), initcheck of the binding
O=gpurun_out/g1c; mkdir -p $O
for i in 1 2; do
  timeout 120 python tools/step_gap.py > $O/gap_chain_$i.txt 2>&1
  DSGD_LT_CHAIN=0 timeout 120 python tools/step_gap.py > $O/gap_nochain_$i.txt 2>&1
  timeout 120 python ab_tmp/r1/step_gap.py > $O/gap_r1_$i.txt 2>&1
done
DSGD_PDL=0 DSGD_LT_CHAIN=0 timeout 120 python tools/step_gap.py > $O/gap_nopdl.txt 2>&1
timeout 900 compute-sanitizer --tool initcheck --print-limit 50 python -m pytest tests/test_reference_binding.py -q -x -k "c1_allreduce and not mu0 and drivers" > $O/initcheck_binding.log 2>&1; echo initcheck=$? >> $O/status.txt
