mkdir -p gpurun_out/q8
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_methods.py -x -q > gpurun_out/q8/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q8/pytest.log
python tools/phases.py C2 > gpurun_out/q8/c2_ga16.json 2>&1
AFN_FSAI_GA=32 python tools/phases.py C2 > gpurun_out/q8/c2_ga32.json 2>&1
timeout 600 python tools/phases.py C5 > gpurun_out/q8/c5_ga16.json 2>&1
AFN_FSAI_GA=32 timeout 600 python tools/phases.py C5 > gpurun_out/q8/c5_ga32.json 2>&1
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/q8/bench.json 2> gpurun_out/q8/bench.err
