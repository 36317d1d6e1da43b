mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "split or sharded" > gpurun_out/r2q_tests.log 2>&1; echo tests rc=$?
