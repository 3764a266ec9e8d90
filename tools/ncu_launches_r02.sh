B="python bench.py --config C2 --steps 2 --warmup 3 --no-extra --no-cpu-baseline --no-parity --no-batch"
$B > gpurun_out/ncu_c2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_C2_sym.csv $B > gpurun_out/ncu_c2.log 2>&1
B4="python bench.py --config C4 --steps 1 --warmup 3 --no-extra --no-cpu-baseline --no-parity --no-batch"
$B4 > gpurun_out/ncu_c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_C4_sym.csv $B4 > gpurun_out/ncu_c4.log 2>&1
python tools/ncu_summary.py launches gpurun_out/r02_launches_C2_sym.csv > gpurun_out/r02_launches_C2_sym.txt
python tools/ncu_summary.py launches gpurun_out/r02_launches_C4_sym.csv > gpurun_out/r02_launches_C4_sym.txt
