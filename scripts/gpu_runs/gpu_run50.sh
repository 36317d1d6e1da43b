mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "muon" > gpurun_out/r2z6_tests.log 2>&1; echo tests rc=$?
