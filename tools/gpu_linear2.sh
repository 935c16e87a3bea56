mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_linear.py -q > gpurun_out/pytest_linear.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_linear.log
python tools/bench_linear.py > gpurun_out/bench_linear.log 2>&1; echo lin=$?; cat gpurun_out/bench_linear.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'], '%.3g rows/s'%d['value'], '%.4f ms'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:linear_kernel -c 3 -o gpurun_out/r1_linear_full python tools/bench_linear.py --steps 1 --warmup 0 > gpurun_out/ncu_linear.log 2>&1; echo ncu=$?
ncu -i gpurun_out/r1_linear_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size > gpurun_out/linear_raw.csv 2>&1; cat gpurun_out/linear_raw.csv | head -8
