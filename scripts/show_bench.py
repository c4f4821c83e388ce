import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
        print(f.split('/')[-1], round(d['value'], 1), round(d['ms_per_step'], 4), {k: round(v, 4) for k, v in d['kernels_ms'].items()},
              'frac', round(d['roofline']['frac'], 3), {k: round(v) for k, v in d['kernel_gbs'].items()}, d['clocks'].get('sm_mhz'))
    except Exception as e:
        print(f, 'ERR', e)
