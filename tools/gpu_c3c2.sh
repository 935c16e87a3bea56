timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_par.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_par.log
for d in 0 1; do BRIDGER_DEEP=$d python tools/explore.py C3 --steps 5 --tag c3_deep$d >> gpurun_out/c3b.jsonl 2>>gpurun_out/c3b.err; done
python tools/explore.py C2 --steps 10 --tag c2 >> gpurun_out/c3b.jsonl 2>>gpurun_out/c3b.err
python tools/explore.py C5 --rows 1000000 --trees 1250 --steps 4 --tag c5 >> gpurun_out/c3b.jsonl 2>>gpurun_out/c3b.err
echo done
