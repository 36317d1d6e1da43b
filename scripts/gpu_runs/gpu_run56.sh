mkdir -p gpurun_out
out=gpurun_out/r2z_stress2.txt
: > $out
for s in 21 22 23 24 25 26 27 28 29 30 31 32; do timeout 900 python scripts/stress.py $s 50 2>&1 | tail -1 >> $out; done
