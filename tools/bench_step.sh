# quick headline-only bench (no extra/cholesky/cpu legs), 3 repeats
for i in 1 2 3; do python bench.py --steps 10 --warmup 3 --no-extra --no-cholesky --no-cpu 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']
print('step %.3f ms cut %d' % (d['value'], d['quality']['cut']), ' '.join('%s=%.3f' % (n, v['ms_per_step']) for n, v in sorted(k.items())))
"; done
