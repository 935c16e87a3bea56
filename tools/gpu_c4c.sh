mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or c4" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/q_tests.log
for sc in 1 0; do
BRIDGER_STREAM_CODES=$sc timeout 300 python bench.py --config C4 --rows 1000000 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c4_$sc.log 2>&1
tail -1 gpurun_out/c4_$sc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 scodes=$sc', d['value'], d['ms_per_step'], r.get('kernel_ms'))"
done
