timeout 700 python -m pytest tests/test_gpu_ep_multirank.py tests/test_gpu_ep.py -x -q > gpurun_out/p4_tests.log 2>&1; tail -2 gpurun_out/p4_tests.log
python tools/ep_projection.py --G 8 > gpurun_out/proj_ov.json 2>gpurun_out/proj_ov.err
python tools/ep_projection.py --G 8 --no-overlap > gpurun_out/proj_noov.json 2>>gpurun_out/proj_ov.err
python tools/ep_projection.py --G 8 --placement blocked > gpurun_out/proj_ov_bl.json 2>>gpurun_out/proj_ov.err
tail -3 gpurun_out/proj_ov.err
