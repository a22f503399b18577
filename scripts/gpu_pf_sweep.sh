# L2 prefetch sweep (window MB x own-range prefetch) on the default bench, plus the parity tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-pf}
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/${T}_tests.log
for cfg in "0 0" "0 1" "32 1" "48 1" "64 1" "96 1"; do
  set -- $cfg
  QS_PF_WINDOW_MB=$1 QS_PF_OWN=$2 timeout 600 python bench.py --sweep 1,16 --no-cpu --steps 10 > gpurun_out/${T}_w$1_o$2.json 2> gpurun_out/${T}_w$1_o$2.err
  python - "$1" "$2" gpurun_out/${T}_w$1_o$2.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
pb = d["per_batch"]
print(f"window={sys.argv[1]}MB own={sys.argv[2]}: B16 qspec {pb['16']['qspec_tok_s']} ms/cycle {pb['16']['ms_per_cycle']} AR16 {pb['16']['w4a16_ar_tok_s']} | B1 ms/AR {pb['1']['ms_per_ar_step']} ms/cycle {pb['1']['ms_per_cycle']} | frac {d['roofline']['frac']}")
PY
done
