mkdir -p gpurun_out
out=gpurun_out/r2z_l2pf2.txt
: > $out
for rep in 1 2 3; do
for d in 4096 0; do
  echo "== PE_DEBUG_GEMM=$d" >> $out
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-large 4 >> $out 2>&1
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py llama3-8b 2 >> $out 2>&1
done
done
