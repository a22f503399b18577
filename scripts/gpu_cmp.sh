# per-step vs persistent forward on the bench workload (no CPU leg)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; T=${TAG:-cmp}
for P in 0 1; do
QSPEC_PERSISTENT=$P timeout 900 python bench.py --no-cpu --sweep 1,16 --steps 20 > gpurun_out/${T}_p$P.json 2> gpurun_out/${T}_p$P.err; echo "persistent=$P rc=$?"; tail -2 gpurun_out/${T}_p$P.err
python - <<PY
import json
d=json.load(open('gpurun_out/${T}_p$P.json'))
print('value',d['value'],'ar',d['w4a16_ar_tokens_per_s'],'acc',d['acceptance_rate'],'e2e',d['e2e']['value'])
for b,v in d['per_batch'].items(): print(' B',b,v)
print(' roof', d['roofline']['achieved'], d['roofline']['frac'])
PY
done
