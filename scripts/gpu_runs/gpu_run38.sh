mkdir -p gpurun_out
out=gpurun_out/r2z_ld64.txt
: > $out
for s in "1024 1024" "gpt2-small"; do PE_DEBUG_GEMM=128 timeout 300 python profiles/phase_timeline.py $s 2>&1 | grep -A4 epilogue >> $out; done
for d in 0 512 0 512; do echo "dbg $d" >> $out; PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1; PE_DEBUG_GEMM=$d timeout 300 python profiles/small_sweep.py >> $out 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "diagonal_bit_exact or gaussian_parity or muon or unaligned or symmetries or small_path" >> $out 2>&1; echo tests rc=$? >> $out
