# re-entry check: smoke, GPU tests, C2 bench line, C2 launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_c2.log
python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?; tail -1 gpurun_out/bench_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1; echo launch=$?
