# Build-time variants x environment variants of the level-0 pass (mgpbd_pass_burst): bash tools/pass_sweep_env.sh "ENV" "FLAGS" ...
ENVV="$1"; shift
for F in "$@"; do
  MGPBD_EXTRA_NVCC_FLAGS="$F" python paper_2505_13390_b200/build.py --force > gpurun_out/build.log 2>&1 || { echo "build '$F' failed" >> gpurun_out/pass_sweep.txt; continue; }
  echo "== '$F'" >> gpurun_out/pass_sweep.txt
  python tools/pass_env.py "" "$ENVV" >> gpurun_out/pass_sweep.txt 2>&1
done
