mkdir -p gpurun_out/pz
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:wc_gemm_kernel|group_zk_kernel|kmv_cut_kernel" -c 4 -o gpurun_out/pz/zk python tools/profile_case.py C3 > gpurun_out/pz/ncu.log 2>&1
ncu -i gpurun_out/pz/zk.ncu-rep --page details --csv > gpurun_out/pz/details.csv 2>&1
