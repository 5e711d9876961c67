ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 66 -c 1 -o gpurun_out/gu_full python scripts/ncu_verify.py 8 3 > gpurun_out/ncu_gu.log 2>&1
ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/verify_launches_r2.csv python scripts/ncu_verify.py 8 3 > gpurun_out/ncu_l.log 2>&1
tail -3 gpurun_out/ncu_gu.log
