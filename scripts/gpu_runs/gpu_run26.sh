mkdir -p gpurun_out
timeout 600 python profiles/appg_debug.py > gpurun_out/r2z_appg_debug.txt 2>&1; echo rc=$?
