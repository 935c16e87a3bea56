#!/usr/bin/env bash
# The GPU-box tasks of this repo, one entry point (run through gpurun, e.g.
#   /usr/local/graft/bin/gpurun --timeout 1200 -- 'bash tools/gpu.sh tests'
# ).  Outputs land in gpurun_out/ (scratch); summaries worth keeping are
# copied to profiles/ by hand (tools/ncu_summary.py).  One ncu per call; the
# command profiled always runs once without ncu first.  compute-sanitizer is
# closed on this pool (profiles/r2_sanitizer_closed.txt): tools/sanitize_cases.py
# runs the same small cases against the oracle instead.
set -u
mkdir -p gpurun_out
task=${1:-help}; shift || true
case "$task" in
  tests)        # every GPU test + the driver's smoke()
    timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
    tail -3 gpurun_out/pytest_gpu.log
    python -c "import __graft_entry__ as g; g.smoke()" ;;
  bench)        # the default bench line, then the ncu launch list of a short run of the same workload
    python bench.py "$@" > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
    S="python bench.py --no-extra --no-gemm --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 0"
    $S > gpurun_out/bench_short.log 2>&1 && \
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $S \
      > gpurun_out/ncu_launches.log 2>&1; echo "ncu rc=$?" ;;
  explore)      # one timed workload under the current BRIDGER_* environment: tools/explore.py ARGS
    python tools/explore.py "$@" ;;
  ncu)          # ncu --set full of kernels matching REGEX in CMD:  tools/gpu.sh ncu REGEX NAME CMD...
    rx=$1; name=$2; shift 2
    "$@" > gpurun_out/${name}_plain.log 2>&1 && \
      ncu --set full --import-source on --clock-control none -k regex:"$rx" -s 2 -c 1 -o gpurun_out/$name "$@" \
      > gpurun_out/${name}_ncu.log 2>&1; echo "ncu rc=$?" ;;
  sweep-c5)     # K4d configurations on the 1250-tree C5 shard (warps x row-block groups, speculation on/off)
    E="python tools/explore.py C5 --rows 1000000 --trees 1250 --steps 4"
    for cfg in "16 2" "12 2" "8 2" "8 4"; do set -- $cfg
      BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 $E --tag w$1b$2 >> gpurun_out/sweep_c5.jsonl
      BRIDGER_SPEC_D=99 BRIDGER_WARPS=$1 BRIDGER_BLOCKS=$2 $E --tag nospec_w$1b$2 >> gpurun_out/sweep_c5.jsonl
    done
    BRIDGER_DEEP=0 $E --tag k4_partials >> gpurun_out/sweep_c5.jsonl ;;
  sweep-bin)    # binning warps on C3
    for w in 16 12 8; do BRIDGER_BIN_WARPS=$w python tools/explore.py C3 --steps 5 --tag binw$w >> gpurun_out/sweep_bin.jsonl; done ;;
  sparse)       # dense K2 vs 2:4-sparse K2s in the staged GEMM pipeline, several row-block sizes
    for mb in 48 256 1024; do for v in gemm_staged gemm_sparse; do
      BRIDGER_GEMM_SCRATCH_MB=$mb python tools/explore.py C2 --variant $v --steps 3 --tag ${v}_$mb >> gpurun_out/sparse.jsonl
    done; done ;;
  sparse-probe) # pin the tcgen05.mma.sp kind::i8 metadata layout
    nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sparse_probe tools/sparse_probe.cu && timeout 60 /tmp/sparse_probe ;;
  variant-table) # per-depth traverse vs GEMM-form throughput -> profiles/variant_table.json
    python tools/variant_table.py && cp profiles/variant_table.json gpurun_out/ ;;
  sanitize-cases) # every kernel family once, checked against the oracle
    python tools/sanitize_cases.py ;;
  *) sed -n '2,9p' "$0"; echo "tasks: tests bench explore ncu sweep-c5 sweep-bin sparse sparse-probe variant-table sanitize-cases" ;;
esac
