mkdir -p gpurun_out
timeout 1800 python profiles/sweep.py > gpurun_out/r2h_sweep.md 2> gpurun_out/r2h_sweep.err; echo sweep rc=$?
