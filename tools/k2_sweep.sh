for v in 0 1 2 3 4 5; do
  RQ_K2_CFG=$v timeout 300 python -m pytest tests/test_gpu_pair_tma.py -x -q 2>&1 | tail -1
  RQ_K2_CFG=$v timeout 300 python bench.py --workload c1 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg $v', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'kernel_ms %.4f'%r['avg_launch_ms'])"
done
