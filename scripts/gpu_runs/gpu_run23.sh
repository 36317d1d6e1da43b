mkdir -p gpurun_out
timeout 1500 python profiles/sweep.py > gpurun_out/r2w_sweep.md 2> gpurun_out/r2w_sweep.err; echo sweep rc=$?
