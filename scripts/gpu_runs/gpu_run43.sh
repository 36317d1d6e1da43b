mkdir -p gpurun_out
out=gpurun_out/r2z_stress.txt
: > $out
for s in 11 12 13 14 15 16; do timeout 900 python scripts/stress.py $s 50 2>&1 | tail -1 >> $out; done
