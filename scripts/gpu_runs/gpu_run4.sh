mkdir -p gpurun_out
set -x
timeout 600 python profiles/appg_margin.py sweep > gpurun_out/r2d_appg_sweep.txt 2>&1; echo probe rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "sweep_sizes or full_llama or fuzz" > gpurun_out/r2d_gputests.log 2>&1; echo tests rc=$?
