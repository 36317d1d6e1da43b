mkdir -p gpurun_out
out=gpurun_out/r2z_band.txt
: > $out
for rep in 1 2 3; do
for b in 16 8; do
  echo "== PE_BAND_MIN=$b" >> $out
  PE_BAND_MIN=$b timeout 300 python profiles/phase_times.py llama3-8b 3 >> $out 2>&1
done
done
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
PE_BAND_MIN=8 timeout 900 ncu --metrics $M --clock-control none -k regex:pe_gemm --launch-skip 3 --launch-count 3 --csv \
    --log-file gpurun_out/r2z_dram_band8.csv python profiles/run_one.py llama3-8b 32 1 5 > /dev/null 2>&1; echo rc=$?
