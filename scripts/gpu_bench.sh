cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-b}
timeout 900 python bench.py $BENCH_ARGS > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
