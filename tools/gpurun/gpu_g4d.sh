# 4-GPU: in-process multicast teardown fix check, reference-binding failure bisection
O=gpurun_out/g4d; mkdir -p $O
export PYTHONFAULTHANDLER=1
for n in 4 3; do for p in pull-gossip all-reduce; do
  timeout 120 python tools/nvlink_profile.py --gpus $n --protocol $p --rounds 5 >> $O/inproc.jsonl 2>> $O/inproc.err
  echo inproc_${p}_n${n}=$? >> $O/status.txt
done; done
K="drivers and (c1_allreduce or async8 or pull8)"
timeout 300 python -m pytest tests/test_reference_binding.py -q -rf -k "$K" > $O/b1_alone.log 2>&1; echo b1_alone=$? >> $O/status.txt
timeout 300 python tools/debug/bind_probe.py torch > $O/b2_torch.log 2>&1; echo b2_torch=$? >> $O/status.txt
timeout 300 python -m pytest tests/test_multigpu.py tests/test_reference_binding.py -q -rf -k "missing_peer or ($K)" > $O/b3_timeout.log 2>&1; echo b3_timeout=$? >> $O/status.txt
timeout 400 python -m pytest tests/test_multigpu.py tests/test_reference_binding.py -q -rf -k "three_ranks or ($K)" > $O/b4_three.log 2>&1; echo b4_three=$? >> $O/status.txt
timeout 400 python -m pytest tests/test_multigpu.py tests/test_reference_binding.py -q -rf -k "(protocols and f64 and default) or ($K)" > $O/b5_proto.log 2>&1; echo b5_proto=$? >> $O/status.txt
timeout 400 python -m pytest tests/test_multigpu.py tests/test_reference_binding.py -q -rf -k "(logistic and f64) or ($K)" > $O/b6_logistic.log 2>&1; echo b6_logistic=$? >> $O/status.txt
