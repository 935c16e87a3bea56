"""Summarise an ncu report (or a launch-list CSV) into a small committed text file.

usage: python tools/ncu_summary.py gpurun_out/X.ncu-rep profiles/X.txt
       python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/launches_X.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def summarize_rep(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        out.append(f"kernel: {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            for h in hdr:
                if h == k or h.endswith("." + k):
                    out.append(f"  {h:90s} {d[h]:>16s} {units[hdr.index(h)]}")
                    break
        # warp-stall sampling: share of all samples per reason (top 8)
        st = {h[len(STALL):]: float(d[h] or 0) for h in hdr
              if h.startswith(STALL) and not h.endswith("not_issued") and d[h] not in ("", "n/a")}
        tot = sum(st.values())
        if tot > 0:
            top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
            out.append("  stall samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))
    return "\n".join(out) + "\n"


def summarize_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0][:90]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        u = r[ix["Metric Unit"]]
        v = v * 1e3 if u == "ms" else v / 1e3 if u == "ns" else v
        tot[name] += v
        cnt[name] += 1
    all_us = sum(tot.values())
    lines = [f"{'kernel':90s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"{k:90s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k]/cnt[k]:10.2f} {100*tot[k]/all_us:5.1f}%")
    return "\n".join(lines) + "\n(cold-cache, serialised ncu launch list: compare shares, not absolutes)\n"


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        text = summarize_launches(sys.argv[2])
        dst = sys.argv[3]
    else:
        text = summarize_rep(sys.argv[1])
        dst = sys.argv[2]
    open(dst, "w").write(text)
    print(text)
