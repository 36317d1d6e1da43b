mkdir -p gpurun_out
# Alg. 4 (restart 3) on one Llama layer: every launch of one call, ncu --set full
PE_RUN_RECT=3 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pe_gemm|pe_expand" \
  -o /tmp/r2p_alg4_full -f python profiles/run_one.py llama3-8b 1 1 5 > gpurun_out/r2p_alg4_ncu.log 2>&1; echo rc=$?
ncu -i /tmp/r2p_alg4_full.ncu-rep --page raw --csv > gpurun_out/r2p_alg4_raw.csv 2>/dev/null
# GPT-2 S set: iteration 2 (gram, poly, update)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pe_gemm --launch-skip 18 --launch-count 3 \
  -o /tmp/r2p_gpt2s_full -f python profiles/run_one.py gpt2-small 12 2 5 > gpurun_out/r2p_gpt2s_ncu.log 2>&1; echo rc=$?
ncu -i /tmp/r2p_gpt2s_full.ncu-rep --page raw --csv > gpurun_out/r2p_gpt2s_raw.csv 2>/dev/null
ls -la gpurun_out
