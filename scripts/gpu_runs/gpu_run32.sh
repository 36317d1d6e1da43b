mkdir -p gpurun_out
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo bench rc=$? wall $(( $(date +%s) - s )) s
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r2z_ref.json 2> gpurun_out/r2z_ref.err; echo ref rc=$? wall $(( $(date +%s) - s )) s
