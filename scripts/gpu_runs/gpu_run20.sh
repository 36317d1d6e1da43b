mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "restart_one or polar_split_peers or two_plane" > gpurun_out/r2t_tests.log 2>&1; echo tests rc=$?
