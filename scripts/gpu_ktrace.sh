# Device timelines of the real decode graphs (scripts/ktrace_step.py) + the GPU tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-kt}
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/${T}_tests.log
fi
timeout 300 python scripts/ktrace_step.py --batch 1 --algorithm greedy --dump gpurun_out/${T}_ar1.json > gpurun_out/${T}_ar1.txt 2>&1; echo "ar1 rc=$?"; cat gpurun_out/${T}_ar1.txt
timeout 300 python scripts/ktrace_step.py --batch 16 --algorithm qspec --dump gpurun_out/${T}_b16.json > gpurun_out/${T}_b16.txt 2>&1; echo "b16 rc=$?"; cat gpurun_out/${T}_b16.txt
