set -x
BENCH="python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline --no-parity --no-batch"
$BENCH > gpurun_out/ncu_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launches_bench_C4.csv $BENCH > gpurun_out/ncu_bench.log 2>&1
for m in 20 10 15 21; do
  python tools/profile_residual.py --m $m > gpurun_out/prof_plain_$m.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bsr_stream_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_residual_m$m python tools/profile_residual.py --m $m > gpurun_out/ncu_res_$m.log 2>&1
done
ls -la gpurun_out/
