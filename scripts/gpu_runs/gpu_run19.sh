mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "diagonal or scale_range or symmetries or gaussian or empty or debug or degree3 or muon or full_llama_set_sampled" > gpurun_out/r2s_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --extra '' --no-cpu-baseline > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo bench rc=$?
