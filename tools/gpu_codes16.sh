mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "coded or c2 or c3 or c5 or pruned" -x > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/q_tests.log
python bench.py --config C2 --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/q_C2.log 2>&1
tail -1 gpurun_out/q_C2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C2', d['value'], d['ms_per_step'], r.get('kernel_ms'))"
