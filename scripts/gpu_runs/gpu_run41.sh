mkdir -p gpurun_out
out=gpurun_out/r2z_slots.txt
: > $out
P=$GRAFT_REPO_ROOT/paper_2505_16932_b200
for rep in 1 2; do
for v in libpe libpe_v1 libpe_v2 libpe_v3; do
  echo "== $v" >> $out
  PE_LIB_OVERRIDE=$P/$v.so timeout 300 python profiles/phase_times.py gpt2-small 10 >> $out 2>&1
  PE_LIB_OVERRIDE=$P/$v.so timeout 300 python profiles/phase_times.py gpt2-large 4 >> $out 2>&1
  PE_LIB_OVERRIDE=$P/$v.so timeout 300 python profiles/phase_times.py llama3-8b 1 >> $out 2>&1
done
done
