# threshold-bin codes experiment: parity tests, timings with codes on/off (C2, C3), ncu of bin + traversal (C2)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "coded or c2 or c3 or pruned or chunk" > gpurun_out/codes_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/codes_tests.log
for cfg in C2 C3; do for c in 0 1; do
  BRIDGER_CODES=$c python bench.py --config $cfg --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/codes_${cfg}_$c.log 2>&1; echo $cfg codes$c=$?
  tail -1 gpurun_out/codes_${cfg}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg codes', $c, d['ms_per_step'], d['roofline']['kernel_ms'])"
done; done
BRIDGER_CODES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bin_kernel|trav_kernel" -c 2 -o gpurun_out/codes_c2 python bench.py --config C2 --no-cpu-baseline --no-gemm --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/codes_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/codes_ncu.log
