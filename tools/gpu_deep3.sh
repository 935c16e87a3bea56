python -m pytest tests -m gpu -x -q -k "parity or fullsize or models" > gpurun_out/pytest_deep3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_deep3.log
E5="python tools/explore.py C5 --rows 1000000 --trees 1250 --steps 4"
for cfg in "16 2" "8 2" "12 2"; do set -- $cfg
BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 $E5 --tag spec_w$1b$2 >> gpurun_out/deep3.jsonl 2>>gpurun_out/deep3.err
BRIDGER_SPEC_D=99 BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 $E5 --tag nospec_w$1b$2 >> gpurun_out/deep3.jsonl 2>>gpurun_out/deep3.err
done
BRIDGER_SPEC_D=6 python tools/explore.py C3 --steps 5 --tag c3_spec >> gpurun_out/deep3.jsonl 2>>gpurun_out/deep3.err
python tools/explore.py C3 --steps 5 --tag c3_nospec >> gpurun_out/deep3.jsonl 2>>gpurun_out/deep3.err
echo done
