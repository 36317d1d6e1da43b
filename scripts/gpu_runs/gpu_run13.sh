mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "diagonal or gaussian or degree3 or small or fuzz or batch or two_plane" > gpurun_out/r2m_tests.log 2>&1; echo tests rc=$?
