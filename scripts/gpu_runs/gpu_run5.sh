mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "alg4" > gpurun_out/r2e_alg4.log 2>&1; echo alg4 rc=$?
timeout 600 python profiles/appg_margin.py sweep > gpurun_out/r2e_appg_sweep.txt 2>&1; echo probe rc=$?
timeout 300 python profiles/appg_margin.py > gpurun_out/r2e_appg_margin.txt 2>&1; echo probe2 rc=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2e_gputests.log 2>&1; echo tests rc=$?
