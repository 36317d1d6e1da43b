mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --extra gpt2-small --no-cpu-baseline > gpurun_out/r2z_bench_q.json 2> gpurun_out/r2z_bench_q.err; echo bench rc=$?
