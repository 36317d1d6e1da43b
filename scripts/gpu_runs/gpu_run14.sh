mkdir -p gpurun_out
for g in 8 16 32 48; do PE_HOST_GROUPS=$g timeout 300 python profiles/e2e_times.py llama3-8b >> gpurun_out/r2n_e2e.txt 2>&1; done
for g in 4 8 12 16; do PE_HOST_GROUPS=$g timeout 120 python profiles/e2e_times.py gpt2-small >> gpurun_out/r2n_e2e.txt 2>&1; done
