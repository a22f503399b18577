cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-mk}
timeout 600 python -m pytest tests/test_gpu_mk.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo "mk tests rc=$?"; tail -30 gpurun_out/${T}_tests.log
timeout 600 python bench.py --no-cpu --sweep 1,16 --steps 20 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -5 gpurun_out/${T}_bench.err
python - <<'PY'
import json,os
T=os.environ.get('TAG','mk')
try:
    d=json.load(open(f'gpurun_out/{T}_bench.json'))
    print('value',d['value'],'ar',d['w4a16_ar_tokens_per_s'],'acc',d['acceptance_rate'])
    print('per_batch',json.dumps(d['per_batch']))
    print('roof', json.dumps(d['roofline'])[:600])
except Exception as e: print('no bench', e)
PY
