# quick: codes parity subset + C2/C3 bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "coded or c2 or c3 or pruned or chunk" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/q_tests.log
for cfg in C2 C3; do
  python bench.py --config $cfg --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/q_$cfg.log 2>&1; echo $cfg=$?
  tail -1 gpurun_out/q_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', d['value'], d['ms_per_step'], r.get('kernel_ms'), r.get('frac'))"
done
