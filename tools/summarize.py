import sys, json
for l in open(sys.argv[1]):
    if l.startswith('ARGS'): print(l.strip()); continue
    try: d = json.loads(l)
    except Exception: continue
    rf = d.get('roofline') or {}
    bb = d.get('busbw')
    print('  value %.4f ms  roof %s %.0f GB/s frac %.2f kern %s busbw %s' % (d['value'], rf.get('kernel'), rf.get('achieved', 0), rf.get('frac', 0), {k: round(v, 4) for k, v in d.get('kernel_ms_per_step', {}).items()}, bb and (round(bb['value']), bb['algo'], round(bb['ms'], 4))))
