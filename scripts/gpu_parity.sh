cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_draft_parity.py -q > gpurun_out/g1_draft.log 2>&1; echo "draft rc=$?"; tail -30 gpurun_out/g1_draft.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/g1_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/g1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/g1_smoke.log
timeout 600 python bench.py --sweep 1,16 --no-cpu --steps 10 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/g1_bench.json
