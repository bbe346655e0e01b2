# Bench under environment-switch variants (same build): bash tools/bench_env.sh "" "MGPBD_NO_TAIL=1" ...
for V in "$@"; do
  env $V python bench.py --no-cpu-baseline > gpurun_out/bench_env.json 2>/dev/null
  V="$V" python -c "
import json, os; d=json.loads(open('gpurun_out/bench_env.json').read().strip().splitlines()[-1]); c=d['config']
print(repr(os.environ['V']), round(d['value'],2), 'steady', round(c['ms_frame_steady_median'],2), 'setups', c['setups_in_window'], 'indef', c['indefinite_events_in_window'], 'L1', c['levels'][1][0], 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" >> gpurun_out/bench_env.txt
done
