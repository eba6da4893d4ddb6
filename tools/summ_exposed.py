import json, sys
for l in open(sys.argv[1]):
    if l.startswith('ARGS'): print(l.strip()); continue
    try: d = json.loads(l)
    except Exception: continue
    e = d.get('exposed')
    bb = d.get('busbw')
    print('   synthetic step %.3f ms kern %s busbw %s' % (d['value'], {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items()}, bb and round(bb['value'])))
    if e:
        t = e['timeline_rank0'] or {}
        print('   exposed: bwd %.2f sync %.2f exposed %.3f ms (%.1f%%) no-overlap exposed %.3f' % (e['t_bwd_ms'], e['t_bwd_plus_sync_ms'], e['exposed_ms'], e['exposed_pct_of_bwd'], e['exposed_no_overlap_ms']))
        if t: print('   timeline: last_ready %.2f last_end %.2f tail %.3f max_queue %.3f busy %.2f n %d' % (t['last_ready_ms'], t['last_end_ms'], t['tail_ms'], t['max_queue_delay_ms'], t['comm_busy_ms'], t['launches']))
        if t.get('per_launch'): print('   ', t['per_launch'][:4], '...', t['per_launch'][-4:])
