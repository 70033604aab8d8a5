import json, sys
for c in sys.argv[1:] or ('c2', 'c3', 'c4'):
    try:
        d = json.loads(open(f'gpurun_out/bench_{c}.json').read().strip().splitlines()[-1])
    except Exception as e:
        print(c, 'ERR', e, open(f'gpurun_out/bench_{c}.json').read()[-2000:]); continue
    print(c, 'ms', round(d['ms_per_step'], 3), 'pairs/s', round(d['value']), 'nnz/pair', round(d['nnz_per_pair']),
          'peakGB', round(d['peak_gb'], 3), 'launches', d['gpu_launches'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
    print('  stages', {k: round(v, 3) for k, v in d['stages_ms'].items()})
    print('  roof', d['roofline']['kernel'], round(d['roofline']['frac'], 3), ' dist', round(d['roofline_distance_pass']['frac'], 3),
          'e2e', d['e2e'] and round(d['e2e']['value']), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'], 1))
