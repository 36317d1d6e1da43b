mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x -k "split_k" > gpurun_out/r2x_tests.log 2>&1; echo tests rc=$?
for k in 1 2 4; do PE_SPLIT_K=$k timeout 300 python profiles/small_sweep.py >> gpurun_out/r2x_small.txt 2>&1; done
