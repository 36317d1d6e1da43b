mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "spectrum_init or graph" > gpurun_out/r2z8_tests.log 2>&1; echo tests rc=$?
timeout 600 python profiles/init_times.py > gpurun_out/r2z_init_times.txt 2>&1; echo times rc=$?
