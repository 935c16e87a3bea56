mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fz_kernel -c 1 -o gpurun_out/fz_c3 python bench.py --config C3 --rows 1000000 --variant gemm --no-cpu-baseline --no-gemm --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/fz_ncu3.log 2>&1; echo ncu=$?
