mkdir -p gpurun_out
out=gpurun_out/r2z_l2pf.txt
: > $out
for rep in 1 2; do
for d in 0 4096; do
  echo "== PE_DEBUG_GEMM=$d" >> $out
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-large 4 >> $out 2>&1
  PE_DEBUG_GEMM=$d timeout 300 python profiles/small_sweep.py >> $out 2>&1
done
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "diagonal_bit_exact or gaussian_parity or unaligned or iteration_counts or alg4_parity" >> $out 2>&1; echo tests rc=$? >> $out
