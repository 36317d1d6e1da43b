mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "alg4" -rf > gpurun_out/r2k_tests.log 2>&1; echo tests rc=$?
PE_FUSED=0 timeout 300 python profiles/small_sweep.py > gpurun_out/r2k_small.txt 2>&1
PE_FUSED=1 timeout 300 python profiles/small_sweep.py >> gpurun_out/r2k_small.txt 2>&1
