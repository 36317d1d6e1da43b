mkdir -p gpurun_out
timeout 300 python profiles/alg4_debug.py sweep > gpurun_out/r2i_alg4_debug.txt 2>&1; echo rc=$?
