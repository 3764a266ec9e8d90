# warp-state / speed-of-light sections of the half-storage pass: bash tools/ncu_stalls.sh C4 [C5@1024 ...]
for c in "$@"; do
  t=${c/@/_}
  BMG_SYM_HALF=1 ncu --section WarpStateStats --section SpeedOfLight --section SchedulerStats --section MemoryWorkloadAnalysis \
      --clock-control none --profile-from-start off -k regex:"bsr_stream_kernel" -c 1 --csv --page raw \
      --log-file gpurun_out/stalls_$t.csv python tools/profile_sym.py $c > gpurun_out/stalls_$t.log 2>&1
done
