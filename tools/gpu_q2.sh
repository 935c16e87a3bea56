timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "host or f64 or stream" > gpurun_out/q_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/q_tests.log
