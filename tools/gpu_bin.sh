timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "binning or coded or c3" > gpurun_out/pytest_bin.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_bin.log
for w in 16 12 8 6 4; do BRIDGER_BIN_WARPS=$w python tools/explore.py C3 --steps 5 --tag c3_binw$w >> gpurun_out/bin.jsonl 2>>gpurun_out/bin.err; done
echo done
