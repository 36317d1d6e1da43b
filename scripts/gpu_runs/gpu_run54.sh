mkdir -p gpurun_out
out=gpurun_out/r2z_init_ab.txt
: > $out
P=$GRAFT_REPO_ROOT/paper_2505_16932_b200
for rep in 1 2; do
  echo "== merged (libpe)" >> $out; timeout 600 python profiles/init_times.py >> $out 2>&1
  echo "== separate (libpe_old)" >> $out; PE_LIB_OVERRIDE=$P/libpe_old.so timeout 600 python profiles/init_times.py >> $out 2>&1
done
