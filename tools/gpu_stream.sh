mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "stream or c5 or pruned" > gpurun_out/st_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/st_pytest.log
timeout 300 python bench.py --config C4 --rows 1000000 --no-cpu-baseline --no-gemm --steps 5 > gpurun_out/st_bench_c4.log 2>&1; echo b4=$?
BRIDGER_STREAM=0 timeout 300 python bench.py --config C4 --rows 1000000 --no-cpu-baseline --no-gemm --steps 5 > gpurun_out/st_bench_c4_old.log 2>&1; echo b4old=$?
python - <<'PY'
import json
for f in ['gpurun_out/st_bench_c4.log','gpurun_out/st_bench_c4_old.log']:
    try:
        l=json.loads(open(f).read().strip().splitlines()[-1]); print(f, l['value'], l['ms_per_step'], l['roofline'].get('frac'), l['roofline'].get('kernel_ms'))
    except Exception as e: print(f, 'ERR', e, open(f).read()[-2000:])
PY
