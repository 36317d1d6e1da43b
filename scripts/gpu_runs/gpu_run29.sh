mkdir -p gpurun_out
out=gpurun_out/r2z_gpt2s_dbg.txt
: > $out
for d in 0 1 8 9 2048 2049 32 33; do
  echo "== PE_DEBUG_GEMM=$d" >> $out
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
done
echo "== stats" >> $out
PE_DEBUG_GEMM=4 timeout 300 python profiles/gemm_stats.py gpt2-small >> $out 2>&1
PE_DEBUG_GEMM=4 timeout 300 python profiles/gemm_stats.py llama3-8b >> $out 2>&1
