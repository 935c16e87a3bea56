E5="python tools/explore.py C5 --rows 1000000 --trees 1250 --steps 4"
for cfg in "16 2" "8 2" "8 4" "12 2"; do set -- $cfg
BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 $E5 --tag deep2_w$1b$2 >> gpurun_out/deep2.jsonl 2>>gpurun_out/deep2.err
done
python tools/explore.py C3 --steps 5 --tag c3_deep2 >> gpurun_out/deep2.jsonl 2>>gpurun_out/deep2.err
echo done
