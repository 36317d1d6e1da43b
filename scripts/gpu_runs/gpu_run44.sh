mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "spectrum_init_diagonal_emulation or no_fold" > gpurun_out/r2z5_tests.log 2>&1; echo tests rc=$?
