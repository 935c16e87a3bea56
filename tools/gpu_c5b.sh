mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "c5 or chunk" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/q_tests.log
run() { tail -1 gpurun_out/$1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['value'], d['ms_per_step'], r.get('kernel_ms'), r.get('frac'))"; }
BRIDGER_DEBUG=1 python bench.py --config C5 --rows 1000000 --trees 1250 --no-cpu-baseline --e2e-steps 0 --steps 3 > gpurun_out/c5.log 2>gpurun_out/c5.err; run c5; grep "trav_kernel mode" gpurun_out/c5.err | tail -1
