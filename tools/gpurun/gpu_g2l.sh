# 2-GPU: EASGD with the gpu-scope round counter -- parity and latency
O=gpurun_out/${OUT:-g2l}; mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu.py tests/test_inproc_ranks.py -q -rf -x -k "default or elastic or missing_peer" > $O/pytest.log 2>&1; echo pytest=$? >> $O/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tools/small_d_probe.py --sizes 4096,1e6,25e6 --protocols elastic-avg > $O/probe.jsonl 2> $O/probe.err; echo probe=$? >> $O/status.txt
