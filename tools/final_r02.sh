# the driver's own commands (reference arm first, then ours), then the launch list of the bench command
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
B="python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline --no-parity --no-batch"
$B > gpurun_out/ncu_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off \
    --csv --log-file gpurun_out/r02_launches_bench_C4.csv $B > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_summary.py launches gpurun_out/r02_launches_bench_C4.csv > gpurun_out/r02_launches_bench_C4.txt
