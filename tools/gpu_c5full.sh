timeout 900 python bench.py --config C5 --rows 200000 --steps 2 --warmup 3 --no-gemm --no-cpu-baseline --e2e-steps 0 > gpurun_out/c5full.log 2>&1; echo c5full=$?
tail -1 gpurun_out/c5full.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c5 full 200k rows', d['value'], d['ms_per_step'], r.get('kernel_ms'), r.get('node_format'), d['exact_tier'])"
