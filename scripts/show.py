import json, sys, subprocess
tag = sys.argv[1]
print(open(f'gpurun_out/{tag}_gpu.txt').read()[-400:])
for l in open(f'gpurun_out/{tag}_bench.txt'):
    if l.startswith('{'):
        d = json.loads(l); r = d['roofline']
        print('value', d['value'], 'ms', d['ms_per_step'], 'ratio', d['ckpt_over_nockpt_time'], 'frac', r['frac'],
              {k: v['avg_us'] for k, v in r['per_kind'].items()}, 'e2e', round(d['e2e']['value'], 1),
              'bitwise', d['nockpt']['bitwise_equal_loss'] if d['nockpt'] else None, 'launches', d['gpu_launches'])
    else:
        print(l[:300].rstrip())
print(open(f'gpurun_out/{tag}_phases.txt').read())
subprocess.run([sys.executable, 'scripts/summ_launch.py', f'gpurun_out/{tag}_launches32.csv'])
