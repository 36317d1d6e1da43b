mkdir -p gpurun_out
out=gpurun_out/r2z_timeline2.txt
: > $out
for d in 128 384; do
for s in "1024 1024" "2048 2048" "gpt2-small"; do echo "dbg $d" >> $out; PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_timeline.py $s >> $out 2>&1; done
done
for d in 0 256 0 256; do echo "dbg $d" >> $out; PE_DEBUG_GEMM=$d timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1; PE_DEBUG_GEMM=$d timeout 300 python profiles/small_sweep.py >> $out 2>&1; done
