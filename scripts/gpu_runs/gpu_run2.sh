mkdir -p gpurun_out
set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "spectrum_init" > gpurun_out/r2b_appg.log 2>&1; echo appg rc=$?
# ncu --set full of iteration 3 (gram, poly, update) of one pe_polar over the full Llama-3-8B set
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pe_gemm --launch-skip 6 --launch-count 3 \
  -o gpurun_out/r2b_llama_full -f python profiles/run_one.py llama3-8b 32 1 5 > gpurun_out/r2b_ncu_full.log 2>&1; echo ncufull rc=$?
ncu -i gpurun_out/r2b_llama_full.ncu-rep --page raw --csv > gpurun_out/r2b_llama_full_raw.csv 2>/dev/null
# launch list of the bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv \
  python bench.py --steps 2 --warmup 1 --extra '' --no-cpu-baseline > gpurun_out/r2b_ncu_bench.log 2>&1; echo launches rc=$?
