for r in 1 2; do for v in 0 1.0 0.6; do HM_L2_PERSIST_X=$v python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras --sustained-steps 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('PERSIST=$v', round(d['value']/1e6,3), {k: round(x,1) for k,x in d['config']['stages_us'].items()})"; done; done
for v in 0 1.0; do HM_L2_PERSIST_X=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:grouped_gemm -s 4 -c 2 --csv --log-file gpurun_out/l2p_$v.csv python bench.py --eager --steps 2 --warmup 3 --no-clocks --no-cpu-baseline --no-extras --sustained-steps 0 > /dev/null 2>&1; grep -h "dram__bytes_read\|duration" gpurun_out/l2p_$v.csv | cut -d, -f5,12-16 | head -6; done
