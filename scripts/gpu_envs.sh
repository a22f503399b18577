#!/bin/bash
# Bench (B=1 / B=16, no CPU arm) under several env settings: ENVS="name1:K=V,K2=V2 name2:..."
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-ev}
for spec in $ENVS; do
  name=${spec%%:*}; kv=${spec#*:}
  env $(echo $kv | tr ',' ' ') timeout 600 python bench.py --sweep ${SWEEP:-1,16} --no-cpu --steps ${STEPS:-10} > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err; echo "== $name ($kv) rc=$?"
  python - gpurun_out/${T}_$name.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
pb=d["per_batch"]
print("value",d["value"],"ar",d["w4a16_ar_tokens_per_s"],"frac",d["roofline"]["frac"],"e2e",d["e2e"]["value"], "launches", d.get("gpu_launches"))
for b,v in pb.items(): print(b, {k: v[k] for k in ("qspec_tok_s","w4a16_ar_tok_s","ms_per_cycle","ms_per_ar_step")})
print("cost", d["cost_model"]["profile_ms"])
PY
done
