for k in 3 7; do
ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2c_verify_b8k${k}_dram.csv python scripts/ncu_verify.py 8 $k > /dev/null 2>&1
done
python scripts/verify_traffic.py gpurun_out/verify_traffic.json 8:3:gpurun_out/r2c_verify_b8k3_dram.csv 8:7:gpurun_out/r2c_verify_b8k7_dram.csv
PB=8 PK=7 ncu --nvtx --nvtx-include "iter/" --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2c_iter_b8k7_launches.csv python scripts/prof_iteration.py > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/r2c_iter_b8k7_launches.csv | tail -14
