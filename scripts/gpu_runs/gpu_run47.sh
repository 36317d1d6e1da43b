mkdir -p gpurun_out
# final build: ncu --set full of iteration 3 (gram, poly, update) of one pe_polar over the Llama-3-8B set
timeout 600 python profiles/run_one.py llama3-8b 32 1 5 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:pe_gemm --launch-skip 6 --launch-count 3 \
  -o /tmp/r2z_llama_full -f python profiles/run_one.py llama3-8b 32 1 5 > gpurun_out/r2z_ncu_full.log 2>&1; echo ncufull rc=$?
ncu -i /tmp/r2z_llama_full.ncu-rep --page raw --csv > gpurun_out/r2z_llama_full_raw.csv 2>/dev/null
# launch list of the bench command
timeout 900 python bench.py --steps 2 --warmup 3 --extra '' --no-cpu-baseline > gpurun_out/r2z_plain_bench.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2z_launches.csv \
  python bench.py --steps 2 --warmup 3 --extra '' --no-cpu-baseline > gpurun_out/r2z_ncu_bench.log 2>&1; echo launches rc=$?
ls -la gpurun_out/r2z_llama_full_raw.csv gpurun_out/r2z_launches.csv
