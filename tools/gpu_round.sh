# full GPU check: smoke, GPU tests, bench lines for C1..C5, launch list + ncu --set full of the C2 bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?
python bench.py --config C1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo c1=$?
python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
python bench.py --config C4 --rows 1000000 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
python bench.py --config C5 --rows 1000000 --trees 1250 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c5s.log 2>&1; echo c5=$?
for f in c2 c1 c3 c4 c5s; do tail -1 gpurun_out/bench_$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$f', d['value'], d['ms_per_step'], r.get('kernel_ms'), r.get('frac'), r.get('node_format'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1; echo launch=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bin_kernel|trav_kernel|trav_combine" -c 3 -o gpurun_out/r1_c2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bin_kernel|trav_kernel" -c 2 -o gpurun_out/r1_c3_full python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/ncu_full3.log 2>&1; echo ncufull3=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"trav_stream|bin_fg" -c 2 -o gpurun_out/r1_c4_full python bench.py --config C4 --rows 1000000 --steps 1 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/ncu_full4.log 2>&1; echo ncufull4=$?
