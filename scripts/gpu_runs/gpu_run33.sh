mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "unaligned or diagonal_bit_exact or alg4_diagonal" > gpurun_out/r2z3_tests.log 2>&1; echo tests rc=$?
