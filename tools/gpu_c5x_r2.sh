E="python tools/explore.py C5 --rows 1000000 --trees 1250 --steps 4"
for cfg in "16 2" "4 2" "4 1" "2 1" "2 2" "8 4" "4 4" "6 2" "6 3"; do set -- $cfg
BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 $E --tag w$1b$2 >> gpurun_out/c5x.jsonl 2>>gpurun_out/c5x.err
done
BRIDGER_WARPS=4 BRIDGER_BLOCKS=4 BRIDGER_XBUDGET=200 $E --tag w4b4x200 >> gpurun_out/c5x.jsonl 2>>gpurun_out/c5x.err
BRIDGER_WARPS=4 BRIDGER_BLOCKS=2 BRIDGER_XBUDGET=64 $E --tag w4b2x64 >> gpurun_out/c5x.jsonl 2>>gpurun_out/c5x.err
$E --tag default > gpurun_out/c5_plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:trav_kernel -s 2 -c 1 -o gpurun_out/r2_c5_trav $E > gpurun_out/c5_ncu.log 2>&1
echo done
