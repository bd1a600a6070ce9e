# GPU test pass (run under gpurun): the -m gpu suite, then smoke(); logs under gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${1:-t}_tests.log 2>&1; echo "tests rc=$?"
tail -25 gpurun_out/${1:-t}_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${1:-t}_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${1:-t}_smoke.log
