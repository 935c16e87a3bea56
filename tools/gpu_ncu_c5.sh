mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"trav_kernel|bin_fg" -c 2 -o gpurun_out/c5_codes python bench.py --config C5 --rows 1000000 --trees 1250 --no-cpu-baseline --no-gemm --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/c5_ncu.log 2>&1; echo ncu=$?
