# Build-time tuning sweep of the level-0 matrix-free pass (GPU box only; rebuilds libmgpbd.so per variant).
# usage: bash tools/sweep_mf_stages.sh "FLAGS_A" "FLAGS_B" ...   -> gpurun_out/sweep.txt
for F in "$@"; do
  MGPBD_EXTRA_NVCC_FLAGS="$F" python paper_2505_13390_b200/build.py --force > gpurun_out/build.log 2>&1 || { echo "build '$F' failed" >> gpurun_out/sweep.txt; continue; }
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>>gpurun_out/err.log | tail -1 | FL="$F" python -c "
import json,os,sys; d=json.loads(sys.stdin.read()); print(repr(os.environ['FL']), round(d['value'],2), 'median', round(d['config']['ms_frame_median'],2), 'frac', round(d['roofline']['frac'],3), 'burst', round(d['roofline_graph_burst']['frac'],3), 'setups', d['config']['setups_in_window'])" >> gpurun_out/sweep.txt
done
