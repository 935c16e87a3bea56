set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm_path.py -x -q > gpurun_out/fz_pytest.log 2>&1; echo pytest=$?
tail -30 gpurun_out/fz_pytest.log
timeout 300 python bench.py --variant gemm --no-cpu-baseline --steps 5 > gpurun_out/fz_bench_c2.log 2>&1; echo b2=$?
tail -c 1500 gpurun_out/fz_bench_c2.log
timeout 300 python bench.py --config C3 --rows 1000000 --variant gemm --no-cpu-baseline --no-gemm --steps 5 > gpurun_out/fz_bench_c3.log 2>&1; echo b3=$?
head -c 400 gpurun_out/fz_bench_c3.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fz_kernel -c 1 -o gpurun_out/fz_c2 python bench.py --variant gemm --no-cpu-baseline --no-gemm --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/fz_ncu.log 2>&1; echo ncu=$?
tail -5 gpurun_out/fz_ncu.log
