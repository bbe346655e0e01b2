# Build-time variants timed on the fixed hierarchies of tools/ab_frames.py: bash tools/ab_build.sh "FLAGS" ... -> gpurun_out/ab_build.txt
for F in "$@"; do
  MGPBD_EXTRA_NVCC_FLAGS="$F" python paper_2505_13390_b200/build.py --force > gpurun_out/build.log 2>&1 || { echo "build '$F' failed" >> gpurun_out/ab_build.txt; continue; }
  echo "== '$F'" >> gpurun_out/ab_build.txt
  python tools/ab_frames.py --resetup-at 2 "" >> gpurun_out/ab_build.txt 2>&1
done
