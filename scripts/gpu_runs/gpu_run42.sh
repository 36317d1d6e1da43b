mkdir -p gpurun_out
out=gpurun_out/r2z_gramst.txt
: > $out
for d in 0 1024 0 1024; do echo "dbg $d" >> $out; PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1; PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-large 4 >> $out 2>&1; done
PE_DEBUG_GEMM=1024 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "gaussian_parity or diagonal_bit_exact" >> $out 2>&1; echo tests rc=$? >> $out
