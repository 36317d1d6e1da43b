mkdir -p gpurun_out
out=gpurun_out/r2z_hint.txt
: > $out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "diagonal_bit_exact or gaussian_parity or unaligned or muon or full_llama" >> $out 2>&1; echo tests rc=$? >> $out
for rep in 1 2; do
for d in 16384 0 ; do
  echo "== PE_DEBUG_GEMM=$d" >> $out
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-large 4 >> $out 2>&1
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py llama3-8b 2 >> $out 2>&1
done
for d in 0 16384 ; do
  echo "== PE_DEBUG_GEMM=$d" >> $out
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-large 4 >> $out 2>&1
  PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py llama3-8b 2 >> $out 2>&1
done
done
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for d in 0 16384; do
  PE_DEBUG_GEMM=$d timeout 600 python profiles/run_one.py llama3-8b 32 1 5 && \
  PE_DEBUG_GEMM=$d timeout 900 ncu --metrics $M --clock-control none -k regex:pe_gemm --launch-skip 3 --launch-count 3 --csv \
    --log-file gpurun_out/r2z_hint_dram_$d.csv python profiles/run_one.py llama3-8b 32 1 5 > /dev/null 2>&1; echo dram $d rc=$? >> $out
done
