mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2z2_tests.log 2>&1; echo tests rc=$?
