timeout 600 python -m pytest tests/test_gpu_gemm_path.py -x -q -k "sparse" > gpurun_out/pytest_sparse.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sparse.log
for mb in 48 256 1024; do for v in gemm_staged gemm_sparse; do
BRIDGER_GEMM_SCRATCH_MB=$mb timeout 300 python tools/explore.py C2 --variant $v --steps 3 --tag c2_${v}_$mb >> gpurun_out/sparse2.jsonl 2>>gpurun_out/sparse2.err
done; done
E="python tools/explore.py C2 --variant gemm_sparse --steps 2"; BRIDGER_GEMM_SCRATCH_MB=48 $E > gpurun_out/p2.log 2>&1 && BRIDGER_GEMM_SCRATCH_MB=48 ncu --set full --import-source on --clock-control none -k regex:"pcs_kernel" -s 20 -c 1 -o gpurun_out/r2_pcs_c2b $E > gpurun_out/ncu_pcs.log 2>&1
echo done
