mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2g_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo smoke rc=$?
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo bench rc=$? wall $(( $(date +%s) - s )) s
