# K4d (trav_deep.cu) parity + timing sweep on one GPU
python -m pytest tests -m gpu -x -q -k "parity or fullsize or models or dist" > gpurun_out/pytest_deep.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_deep.log
E5="python tools/explore.py C5 --rows 1000000 --trees 1250 --steps 4"
for cfg in "16 2" "16 4" "8 2" "8 4" "4 4" "16 1"; do set -- $cfg
BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 $E5 --tag deep_w$1b$2 >> gpurun_out/deep.jsonl 2>>gpurun_out/deep.err
done
BRIDGER_DEEP=0 $E5 --tag old >> gpurun_out/deep.jsonl 2>>gpurun_out/deep.err
python tools/explore.py C3 --steps 5 --tag c3_deep >> gpurun_out/deep.jsonl 2>>gpurun_out/deep.err
BRIDGER_DEEP=0 python tools/explore.py C3 --steps 5 --tag c3_old >> gpurun_out/deep.jsonl 2>>gpurun_out/deep.err
python tools/explore.py C2 --steps 10 --tag c2_deep >> gpurun_out/deep.jsonl 2>>gpurun_out/deep.err
BRIDGER_DEEP=0 python tools/explore.py C2 --steps 10 --tag c2_old >> gpurun_out/deep.jsonl 2>>gpurun_out/deep.err
echo done
