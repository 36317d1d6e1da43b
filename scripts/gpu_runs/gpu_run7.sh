mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "spectrum_init or sharded or alg4" > gpurun_out/r2g_tests.log 2>&1; echo tests rc=$?
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo bench rc=$?
