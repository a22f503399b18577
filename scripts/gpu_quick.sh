#!/bin/bash
# Quick GPU check: linear sweep (C4 subset), GPU tests, short bench (B=1,16).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-q}
timeout 300 python scripts/linear_bench.py --shapes ${SHAPES:-28672x8192,12288x4096,4096x11008} --ms ${MS:-1,4,16,64} --reps 20 > gpurun_out/${T}_lin.jsonl 2>&1; echo "lin rc=$?"
python - gpurun_out/${T}_lin.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: r=json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(f"{r['shape']:>11} M={r['M']:>3} {r['mode']:>5}: lin {r['us_linear_only']:8.2f} us {r['GBps_linear_only']:7.1f} GB/s | pack+lin {r['us']:8.2f}")
PY
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/${T}_tests.log
fi
if [ -z "$NOBENCH" ]; then
timeout 600 python bench.py --sweep 1,16 --no-cpu --steps 10 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python - gpurun_out/${T}_bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
pb=d["per_batch"]
print("value",d["value"],"ar",d["w4a16_ar_tokens_per_s"],"frac",d["roofline"]["frac"],"e2e",d["e2e"]["value"], "prefill", d.get("prefill"))
for b,v in pb.items(): print(b, v)
print("cost", d["cost_model"]["profile_ms"])
print({k:(v.get("GBps"),v["avg_us"]) for k,v in d["roofline"]["per_kind"].items()})
PY
fi
