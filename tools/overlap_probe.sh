for t in 4 8 12 16; do echo "HM_PUSH_TPCS=$t"; HM_PUSH_TPCS=$t python tools/overlap_probe.py 2>&1 | grep "push\|FFN1"; done
python -m pytest tests/test_gpu_ep.py -q -x -k ordered 2>&1 | tail -2
