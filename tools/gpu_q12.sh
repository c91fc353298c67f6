mkdir -p gpurun_out/q12
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "build or pcg or c2" > gpurun_out/q12/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q12/pytest.log
for bc in 2 4; do AFN_FSAI_BC=$bc python tools/phases.py C2 > gpurun_out/q12/c2_bc$bc.json 2>&1; AFN_FSAI_BC=$bc python tools/phases.py C2 >> gpurun_out/q12/c2_bc$bc.json 2>&1; done
AFN_FSAI_BC=4 timeout 600 python tools/phases.py C3 > gpurun_out/q12/c3_bc4.json 2>&1
AFN_FSAI_BC=2 timeout 600 python tools/phases.py C3 > gpurun_out/q12/c3_bc2.json 2>&1
