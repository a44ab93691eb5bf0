import json,sys
for line in sys.stdin:
    if line.startswith('{'):
        d=json.loads(line); print({k:v for k,v in d.items() if k!='units'})
        us=d['units']
        for u in us[4:15]:
            print(u['u'], 'ready', u['ready'], 'pub_med', u['published'], 'pub_max', u['published_max'], 'poll_exit', u['poll_exit'], 'factor', u['factor'], 'lat_after_last', round(u['factor']-u['published_max'],2))
        import statistics
        print('cadence', round((us[14]['ready']-us[4]['ready'])/10,2), 'mean lat_after_last', round(statistics.mean(u['factor']-u['published_max'] for u in us[4:15]),2))
    else: print(line.strip())
