mkdir -p gpurun_out
for s in 1 2 3 4; do timeout 900 python scripts/stress.py $s 60 >> gpurun_out/r2u_stress.txt 2>&1; done
