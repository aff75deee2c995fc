set -x
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_step_launches.csv python tools/one_step.py c4 > gpurun_out/r2_c4_step.log 2>&1; echo "launch list rc=$?"
tail -2 gpurun_out/r2_c4_step.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -c 2 -o gpurun_out/r2_gemm_2M python tools/gemm_ncu_probe.py 2097152 1024 > gpurun_out/r2_gemm_2M.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/r2_gemm_2M.log
