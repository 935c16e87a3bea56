mkdir -p gpurun_out
run() { tail -1 gpurun_out/$1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', d['ms_per_step'], r.get('kernel_ms'))"; }
for cfg in "16 2 120" "8 2 120" "12 2 120" "16 4 144" "16 1 120" "8 1 120"; do set -- $cfg
BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 BRIDGER_XBUDGET=$3 python bench.py --config C5 --rows 1000000 --trees 1250 --no-cpu-baseline --no-gemm --e2e-steps 0 --steps 3 > gpurun_out/c5_$1_$2_$3.log 2>&1; run c5_$1_$2_$3
done
