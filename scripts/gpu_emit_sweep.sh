# Fused-emit variants (QS_EMIT mask) on the default bench's B=1 / B=16 numbers.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-es}
for m in ${MASKS:-0 1 2 3}; do
  QS_EMIT=$m timeout 600 python bench.py --sweep 1,16 --no-cpu --steps 10 > gpurun_out/${T}_m$m.json 2> gpurun_out/${T}_m$m.err
  python - $m gpurun_out/${T}_m$m.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
pb = d["per_batch"]
print(f"emit={sys.argv[1]}: B16 {pb['16']['qspec_tok_s']} tok/s ms/cycle {pb['16']['ms_per_cycle']} AR16 {pb['16']['w4a16_ar_tok_s']} | B1 ms/AR {pb['1']['ms_per_ar_step']} ms/cycle {pb['1']['ms_per_cycle']} | launches {d['gpu_launches']}")
PY
done
