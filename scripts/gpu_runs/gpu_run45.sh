mkdir -p gpurun_out
out=gpurun_out/r2z_epi16.txt
: > $out
for rep in 1 2; do
for e in 0 1; do
  echo "== PE_EPI16=$e" >> $out
  PE_EPI16=$e timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
  PE_EPI16=$e timeout 300 python profiles/phase_times.py gpt2-large 4 >> $out 2>&1
  PE_EPI16=$e timeout 300 python profiles/phase_times.py llama3-8b 1 >> $out 2>&1
  PE_EPI16=$e timeout 300 python profiles/small_sweep.py >> $out 2>&1
done
done
PE_EPI16=1 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "diagonal_bit_exact or gaussian_parity or unaligned or symmetries or iteration_counts or full_gpt2" >> $out 2>&1; echo tests rc=$? >> $out
