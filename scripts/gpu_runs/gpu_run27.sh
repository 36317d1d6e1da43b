mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/r2z_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo smoke rc=$?
