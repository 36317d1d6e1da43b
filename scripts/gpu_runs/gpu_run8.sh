mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/r2h_gputests.log 2>&1; echo tests rc=$?
