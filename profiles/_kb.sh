python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in int dmma; do CKKS_BCONV=$v python profiles/kbench.py 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('variant','$v', d['keyswitch_us'], d['keyswitch_kernels']['bconv'])"; done
python bench.py --no-cpu-baseline --lanes 8 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('boot', d['ms_per_step'], d['roofline']['kernels']['bconv'])"
