# ncu --set full of the full-storage residual pass per BASELINE block size (m = 10 C2 fine,
# 15 C5 shape, 20 C4 fine, 21 C3 shape): exported as raw CSV + details text, reports deleted
# (gpurun_out is capped at 64 MiB)
for m in 20 15 21 10; do
  BMG_SYM_HALF=0 python tools/profile_residual.py --m $m > gpurun_out/prof_plain_$m.log 2>&1 && \
  BMG_SYM_HALF=0 ncu --set full --clock-control none --import-source on -k regex:bsr_stream_kernel -s 2 -c 1 \
      -o gpurun_out/r02_ncu_residual_m$m python tools/profile_residual.py --m $m > gpurun_out/ncu_res_$m.log 2>&1
  ncu -i gpurun_out/r02_ncu_residual_m$m.ncu-rep --page raw --csv > gpurun_out/r02_ncu_residual_m${m}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02_ncu_residual_m$m.ncu-rep --page details > gpurun_out/r02_ncu_residual_m${m}_details.txt 2>/dev/null
  rm -f gpurun_out/r02_ncu_residual_m$m.ncu-rep
done
du -sh gpurun_out
