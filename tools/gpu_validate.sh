set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2a_gputests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2a_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2a_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench exit $?" >> gpurun_out/r2a_bench.err
tail -3 gpurun_out/r2a_gputests.log; tail -2 gpurun_out/r2a_smoke.log; cut -c1-600 gpurun_out/r2a_bench.json
