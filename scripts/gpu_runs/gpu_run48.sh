mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for o in alt fwd; do
  PE_ORDER=$o timeout 600 python profiles/run_one.py llama3-8b 32 1 5 && \
  PE_ORDER=$o timeout 900 ncu --metrics $M --clock-control none -k regex:pe_gemm --launch-skip 0 --launch-count 9 --csv \
    --log-file gpurun_out/r2z_dram_$o.csv python profiles/run_one.py llama3-8b 32 1 5 > /dev/null 2>&1; echo $o rc=$?
done
