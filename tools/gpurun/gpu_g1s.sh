# 1-GPU: compute-sanitizer memcheck / racecheck / synccheck on the new kernels and the binding;
# the reference arm on every host thread
O=gpurun_out/${OUT:-g1s}; mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_reference_binding.py -q -x -k "resident or drivers" > $O/memcheck_binding.log 2>&1; echo memcheck_binding=$? >> $O/status.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_inproc_ranks.py -q -x -k "staged_sizes and (elastic or pull)" > $O/memcheck_inproc.log 2>&1; echo memcheck_inproc=$? >> $O/status.txt
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_inproc_ranks.py -q -x -k "p8_staged_sizes and elastic and f32" > $O/racecheck_ea.log 2>&1; echo racecheck_ea=$? >> $O/status.txt
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_inproc_ranks.py -q -x -k "p8_staged_sizes and elastic and f32" > $O/synccheck_ea.log 2>&1; echo synccheck_ea=$? >> $O/status.txt
timeout 600 python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err; echo ref=$? >> $O/status.txt
