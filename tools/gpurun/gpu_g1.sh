mkdir -p gpurun_out/g1
nvidia-smi > gpurun_out/g1/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs -x > gpurun_out/g1/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/g1/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1; echo smoke=$? >> gpurun_out/g1/status.txt
timeout 400 python bench.py > gpurun_out/g1/bench_n1.json 2> gpurun_out/g1/bench_n1.err; echo n1=$? >> gpurun_out/g1/status.txt
timeout 400 python bench.py --impl reference > gpurun_out/g1/bench_ref_n1.json 2> gpurun_out/g1/bench_ref_n1.err; echo ref=$? >> gpurun_out/g1/status.txt
