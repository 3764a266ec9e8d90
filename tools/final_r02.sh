# Round-2 evidence run on one B200: GPU tests, the driver's own bench commands (reference arm first, then ours),
# the launch list of the bench command, ncu --set full of the half-storage pass (C2, C4) and the traffic JSON.
python -m pytest tests -m gpu -q > gpurun_out/r02_gputest.log 2>&1; tail -2 gpurun_out/r02_gputest.log
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
B="python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline --no-parity --no-batch"
$B > gpurun_out/ncu_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off \
    --csv --log-file gpurun_out/r02_launches_bench_C4.csv $B > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_summary.py launches gpurun_out/r02_launches_bench_C4.csv > gpurun_out/r02_launches_bench_C4.txt
bash tools/ncu_sym_r02.sh > gpurun_out/ncu_sym_r02.log 2>&1
rm -f gpurun_out/*.ncu-rep gpurun_out/*_source.csv
python tools/traffic_from_raw.py residual_m20_sym=gpurun_out/r02_ncu_sym_C4_raw.csv:gpurun_out/prof_sym_plain_C4.log \
    residual_m10_sym=gpurun_out/r02_ncu_sym_C2_raw.csv:gpurun_out/prof_sym_plain_C2.log > gpurun_out/r02_traffic.json
python tools/stall_summary.py gpurun_out/r02_ncu_sym_C4_raw.csv gpurun_out/r02_ncu_sym_C2_raw.csv > gpurun_out/r02_ncu_sym_stalls.txt 2>&1
ls -la gpurun_out | tail -30
