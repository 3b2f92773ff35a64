python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 0 1; do CKKS_PDL=$v python bench.py --no-cpu-baseline --lanes 8 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('boot pdl',$v, d['ms_per_step'], d['e2e']['ms_per_step'], d['precision_log2_max_err'])"; done
for v in 0 1; do CKKS_PDL=$v python profiles/kbench.py 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ks pdl',$v, d['keyswitch_us'], d['ntt_fwd_R48'], d['ntt_inv_R24'])"; done
