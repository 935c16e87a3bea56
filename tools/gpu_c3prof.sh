E="python tools/explore.py C3 --steps 2"
for d in 0 1; do BRIDGER_DEEP=$d python tools/explore.py C3 --steps 5 --tag c3_deep$d >> gpurun_out/c3.jsonl 2>>gpurun_out/c3.err; done
$E > gpurun_out/c3p.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"bin_coop|trav_deep" -s 4 -c 2 -o gpurun_out/r2_c3_step $E > gpurun_out/ncu_c3.log 2>&1
python tools/variant_table.py > gpurun_out/variant_table.log 2>&1; cp profiles/variant_table.json gpurun_out/variant_table.json
echo done
