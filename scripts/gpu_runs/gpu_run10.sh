mkdir -p gpurun_out
timeout 300 python profiles/alg4_debug.py > gpurun_out/r2j_alg4_debug.txt 2>&1; echo rc=$?
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "alg4 or debug_nonfinite" -rf > gpurun_out/r2j_tests.log 2>&1; echo tests rc=$?
