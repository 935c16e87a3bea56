mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:linear_kernel -c 1 -o gpurun_out/r1_linear_softmax python tools/bench_linear.py --steps 1 --warmup 0 --only Softmax > gpurun_out/ncu_linear3.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:linear_kernel -c 1 -o gpurun_out/r1_linear_c3 python tools/bench_linear.py --steps 1 --warmup 0 --only LinReg > gpurun_out/ncu_linear4.log 2>&1; echo ncu=$?
