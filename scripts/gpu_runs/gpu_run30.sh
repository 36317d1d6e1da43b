mkdir -p gpurun_out
out=gpurun_out/r2z_gpt2s_dbg2.txt
: > $out
for d in 0 2 34 16 18; do
  echo "== PE_DEBUG_GEMM=$d" >> $out
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
done
echo "== stats dbg 2" >> $out
PE_DEBUG_GEMM=6 timeout 300 python profiles/gemm_stats.py gpt2-small >> $out 2>&1
