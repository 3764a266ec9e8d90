# ncu --set full of the finest-level residual pass in the symmetric-half form on the C5 and C3 shapes (m = 15, 21)
for c in C5@1024 C3@512; do
  t=${c/@/_}
  BMG_SYM_HALF=1 python tools/profile_sym.py $c > gpurun_out/prof_sym_plain_$t.log 2>&1 && \
  BMG_SYM_HALF=1 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:"bsr_stream_kernel|sym_merge_kernel" -c 2 -o gpurun_out/r02_ncu_sym_$t \
      python tools/profile_sym.py $c > gpurun_out/ncu_sym_$t.log 2>&1
  ncu -i gpurun_out/r02_ncu_sym_$t.ncu-rep --page raw --csv > gpurun_out/r02_ncu_sym_${t}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r02_ncu_sym_$t.ncu-rep --page details > gpurun_out/r02_ncu_sym_${t}_details.txt 2>/dev/null
  rm -f gpurun_out/r02_ncu_sym_$t.ncu-rep
  tail -1 gpurun_out/prof_sym_plain_$t.log
done
