import json, sys
for l in open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/tune_ops.jsonl'):
    d = json.loads(l); r = d['r']
    print({k: v for k, v in d.items() if k != 'r'}, r.get('variant'), r.get('sigma'), r['kernel_ms'],
          r['frac_of_peak'], r.get('sorted', r.get('golden_ok')))
