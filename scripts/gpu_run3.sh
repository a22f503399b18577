cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-x}
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
timeout 900 python bench.py --no-cpu --sweep 1,16 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/${T}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${T}_bench.json'))
print('value',d['value'],'ar',d['w4a16_ar_tokens_per_s'],'speedup',d['speedup_vs_w4a16_ar'],'acc',d['acceptance_rate'])
print('per_batch',json.dumps(d['per_batch']))
r=d['roofline']; print('roof', r['achieved'], r['frac'], r['avg_launch_us'], r['linear_share_ms_per_step'])
print(json.dumps(r['per_kind']))
print('e2e', d['e2e'])
"
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python scripts/profile_step.py --batch 16 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_ar1.csv python scripts/profile_step.py --batch 1 --algorithm greedy > /dev/null 2>&1; echo "ncu2 rc=$?"
