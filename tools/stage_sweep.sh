# k_local_tma at N = 1: staging depth x CTAs per SM, interleaved repeats
mkdir -p gpurun_out/st2
for rep in 1 2; do
  for cfg in "3 1" "3 0" "2 0" "2 1" "4 1" "5 1"; do
    set -- $cfg
    DSGD_LT_STAGES=$1 DSGD_LT_CTAS=$2 timeout 200 python bench.py --no-extras --no-cpu --steps 50 > gpurun_out/st2/n1_s$1_c$2_r$rep.json 2>/dev/null
  done
done
