mkdir -p gpurun_out
timeout 300 python profiles/run_one.py gpt2-small 12 2 5 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pe_gemm --launch-skip 20 --launch-count 1 \
  -o /tmp/r2z_upd -f python profiles/run_one.py gpt2-small 12 2 5 > gpurun_out/r2z_upd_ncu.log 2>&1; echo rc=$?
ncu -i /tmp/r2z_upd.ncu-rep --page source --csv > gpurun_out/r2z_upd_source.csv 2>/dev/null
ncu -i /tmp/r2z_upd.ncu-rep --page raw --csv > gpurun_out/r2z_upd_raw.csv 2>/dev/null
ls -la gpurun_out/r2z_upd*
