mkdir -p gpurun_out
out=gpurun_out/r2z_timeline4.txt
: > $out
for s in "1024 1024" "2048 2048" "gpt2-small"; do PE_DEBUG_GEMM=128 timeout 300 python profiles/phase_timeline.py $s >> $out 2>&1; done
