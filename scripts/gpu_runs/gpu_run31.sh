mkdir -p gpurun_out
out=gpurun_out/r2z_direct.txt
: > $out
for d in 0 64 0 64; do
  echo "== PE_DEBUG_GEMM=$d" >> $out
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
done
PE_DEBUG_GEMM=4 timeout 300 python profiles/gemm_stats.py gpt2-small >> $out 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "diagonal_bit_exact or gaussian_parity or muon or unaligned or symmetries" >> $out 2>&1; echo tests rc=$? >> $out
