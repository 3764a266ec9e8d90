# ncu --set full of the finest-level residual pass, symmetric-half form forced (C2: m = 10, C4: m = 20)
for c in C2 C4; do
  BMG_SYM_HALF=1 python tools/profile_sym.py $c > gpurun_out/prof_sym_plain_$c.log 2>&1 && \
  BMG_SYM_HALF=1 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"bsr_stream_kernel|sym_merge_kernel" -c 4 -o gpurun_out/r02_ncu_sym_$c \
      python tools/profile_sym.py $c > gpurun_out/ncu_sym_$c.log 2>&1
  ncu -i gpurun_out/r02_ncu_sym_$c.ncu-rep --page raw --csv > gpurun_out/r02_ncu_sym_${c}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02_ncu_sym_$c.ncu-rep --page details > gpurun_out/r02_ncu_sym_${c}_details.txt 2>/dev/null
  ncu -i gpurun_out/r02_ncu_sym_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_ncu_sym_${c}_source.csv 2>/dev/null
done
ls -la gpurun_out/ | grep r02_ncu
du -sh gpurun_out
