mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "stream or c4" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/q_tests.log
for b in 1 0; do
BRIDGER_BULK_LEAF=$b python bench.py --config C4 --rows 1000000 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c4_$b.log 2>&1
tail -1 gpurun_out/c4_$b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 bulk=$b', d['value'], d['ms_per_step'], r.get('kernel_ms'))"
done
