import json, sys
t = sys.argv[1]
import os
d = os.path.join(os.path.dirname(__file__), '..', 'gpurun_out')
print(open(f'{d}/{t}_pytest.txt').read().strip().splitlines()[-1])
for l in open(f'{d}/{t}_bounds.txt'):
    name, _, js = l.partition(' {')
    try:
        r = json.loads('{' + js)
        print(name, r['chunk16']['us'], r['chunk16']['tflops'])
    except Exception:
        print(l[:300])
try:
    tr = json.loads(open(f'{d}/{t}_trace.txt').read().strip().splitlines()[-1])
    for k in ('softmax_A', 'softmax_B', 'mma'):
        print(' ', k, tr[k])
except Exception as e:
    print('trace:', e)
try:
    b = json.loads(open(f'{d}/{t}_bench.txt').read().strip().splitlines()[-1])
    print('bench', b['value'], b['roofline']['per_launch_us'], b['clocks'])
except Exception as e:
    print('bench:', e)
