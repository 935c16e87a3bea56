mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:trav_stream -c 1 -o gpurun_out/c4_stream python bench.py --config C4 --rows 1000000 --no-cpu-baseline --no-gemm --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/c4_ncu.log 2>&1; echo ncu=$?
tail -2 gpurun_out/c4_ncu.log | cut -c1-200
