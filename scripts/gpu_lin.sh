cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-l}
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
timeout 600 python scripts/linear_bench.py --shapes 11008x4096,4096x11008 > gpurun_out/${TAG}_lin.jsonl 2>&1; echo "lin rc=$?"
cat gpurun_out/${TAG}_lin.jsonl
