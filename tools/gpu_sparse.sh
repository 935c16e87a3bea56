timeout 600 python -m pytest tests/test_gpu_gemm_path.py -x -q > gpurun_out/pytest_sparse.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sparse.log
for v in gemm_staged gemm_sparse; do
timeout 300 python tools/explore.py C2 --variant $v --steps 3 --tag c2_$v >> gpurun_out/sparse.jsonl 2>>gpurun_out/sparse.err
timeout 300 python tools/explore.py C2 --variant $v --trees 100 --rows 1000000 --steps 3 --tag c2b_$v >> gpurun_out/sparse.jsonl 2>>gpurun_out/sparse.err
done
echo done
