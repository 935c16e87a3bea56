mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "coded or c5" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/q_tests.log
run() { tail -1 gpurun_out/$1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['value'], d['ms_per_step'], r.get('kernel_ms'), r.get('frac'), r.get('node_format'))"; }
BRIDGER_CODES=0 python bench.py --config C5 --rows 1000000 --trees 1250 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c5_fp32.log 2>&1; run c5_fp32
for xb in 120 144; do
BRIDGER_XBUDGET=$xb python bench.py --config C5 --rows 1000000 --trees 1250 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c5_codes_$xb.log 2>&1; run c5_codes_$xb
BRIDGER_XBUDGET=$xb python bench.py --config C3 --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/c3_codes_$xb.log 2>&1; run c3_codes_$xb
done
