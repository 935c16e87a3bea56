# capture ncu summaries on the box (the .ncu-rep files are large: summarised there, then deleted)
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench_c2.log 2>&1; echo bench=$?
python bench.py --config C4 --rows 1000000 --no-cpu-baseline --e2e-steps 0 > gpurun_out/prof/bench_c4.log 2>&1; echo c4=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > /dev/null 2>&1; echo launch=$?
python tools/ncu_summary.py --launches gpurun_out/prof/launches_c2.csv gpurun_out/prof/r1_launches_c2_codes.txt > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bin_kernel|trav_kernel|trav_combine" -c 3 -o /tmp/r1_c2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > /dev/null 2>&1; echo ncu2=$?
python tools/ncu_summary.py /tmp/r1_c2_full.ncu-rep gpurun_out/prof/r1_codes_c2_ncu_full.txt > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"trav_stream|bin_fg" -c 2 -o /tmp/r1_c4_full python bench.py --config C4 --rows 1000000 --steps 1 --warmup 3 --no-cpu-baseline --no-gemm --e2e-steps 0 > /dev/null 2>&1; echo ncu4=$?
python tools/ncu_summary.py /tmp/r1_c4_full.ncu-rep gpurun_out/prof/r1_stream_codes_c4_ncu_full.txt > /dev/null
ncu -i /tmp/r1_c4_full.ncu-rep --page source --csv --print-source sass -k regex:trav_stream -c 1 > /tmp/c4src.csv 2>/dev/null
python - <<'PY' > gpurun_out/prof/r1_stream_codes_c4_stalls.txt
import csv, collections
rows=list(csv.reader(open('/tmp/c4src.csv')))
h=rows[1]; ix={k:i for i,k in enumerate(h)}
st=collections.Counter()
for r in rows[2:]:
    if len(r)!=len(h) or r[0]=="Address": continue
    for k in h:
        if k.startswith('stall_') and '(Not Issued)' not in k:
            try: st[k]+=int(r[ix[k]] or 0)
            except: pass
t=sum(st.values()) or 1
print("trav_stream_kernel (codes, C4 1M rows) warp-stall sampling shares:")
for k,v in st.most_common(10): print(f"  {k:28s} {100*v/t:5.1f}%")
PY
ls -la gpurun_out/prof
