mkdir -p gpurun_out
out=gpurun_out/r2z_notl.txt
: > $out
for i in 1 2; do PE_DEBUG_GEMM=0 timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1; timeout 300 python profiles/small_sweep.py >> $out 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "diagonal_bit_exact or gaussian_parity or muon or unaligned or symmetries or small_path or stats or debug" >> $out 2>&1; echo tests rc=$? >> $out
