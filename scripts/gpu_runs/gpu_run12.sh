mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "diagonal or gaussian or degree3 or small or fuzz or iteration_counts or symmetries or edges or power_law or batch" > gpurun_out/r2l_tests.log 2>&1; echo tests rc=$?
PE_SMALL_PLANES=1 timeout 300 python profiles/small_times.py > gpurun_out/r2l_small_times.txt 2>&1
PE_SMALL_PLANES=2 timeout 300 python profiles/small_times.py >> gpurun_out/r2l_small_times.txt 2>&1
