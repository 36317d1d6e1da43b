mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "spectrum_init or polar_ex" > gpurun_out/r2z7_tests.log 2>&1; echo tests rc=$?
