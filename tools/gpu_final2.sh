export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f2_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/f2_gputests.log; tail -2 gpurun_out/f2_gputests.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f2_bench_ref.json 2> gpurun_out/f2_bench_ref.err; echo "ref exit $?"; tail -c 400 gpurun_out/f2_bench_ref.json
