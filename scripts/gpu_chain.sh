#!/bin/bash
# Chained-launch check: emit/chain bit-identity tests first (fail fast), then the GPU
# suite, then the B=1 / B=16 bench with chains on (default) and off (QS_EMIT=3).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-ch}
timeout 300 python -m pytest tests/test_gpu_emit.py -x -q > gpurun_out/${T}_emit.log 2>&1; echo "emit rc=$?"; tail -15 gpurun_out/${T}_emit.log
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/${T}_tests.log
fi
for m in ${MASKS:-7 3}; do
QS_EMIT=$m timeout 600 python bench.py --sweep 1,16 --no-cpu --steps 10 > gpurun_out/${T}_m$m.json 2> gpurun_out/${T}_m$m.err; echo "bench m$m rc=$?"
python - gpurun_out/${T}_m$m.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
pb=d["per_batch"]
print("value",d["value"],"ar",d["w4a16_ar_tokens_per_s"],"frac",d["roofline"]["frac"],"e2e",d["e2e"]["value"], "launches", d.get("gpu_launches"))
for b,v in pb.items(): print(b, {k: v[k] for k in ("qspec_tok_s","w4a16_ar_tok_s","ms_per_cycle","ms_per_ar_step")})
print("cost", d["cost_model"]["profile_ms"])
print({k:(v.get("GBps"),v["avg_us"]) for k,v in d["roofline"]["per_kind"].items()})
PY
done
