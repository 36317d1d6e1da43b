mkdir -p gpurun_out
set -x
timeout 300 python profiles/appg_margin.py > gpurun_out/r2c_appg_margin.txt 2>&1; echo probe rc=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c_gputests.log 2>&1; echo tests rc=$?
