for rep in 1 2 3; do for cfg in "32 2" "16 2" "24 2" "12 2"; do set -- $cfg
BRIDGER_H2D_MB=$1 BRIDGER_H2D_STAGES=$2 python bench.py --no-cpu-baseline --no-gemm --steps 3 --e2e-steps 10 > gpurun_out/e2e_$1_$2.log 2>&1
tail -1 gpurun_out/e2e_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mb=$1 st=$2', d['e2e']['value'])"
done; done
