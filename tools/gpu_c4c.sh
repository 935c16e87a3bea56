mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or c4" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/q_tests.log
for w in 3 2; do
BRIDGER_STREAM_W=$w timeout 300 python bench.py --config C4 --rows 1000000 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c4_$w.log 2>&1
tail -1 gpurun_out/c4_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c4 W=$w', d['value'], d['ms_per_step'], r.get('kernel_ms'))"
done
