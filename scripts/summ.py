import json,sys,glob
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); r=d.get('roofline',{})
            print(f.split('/')[-1], round(d['value']), 'ms/step', round(d['ms_per_step']*1000,1),'us kern_us', round(r.get('kernel_ms_mean',0)*1000,1), 'GB/s', round(r.get('achieved',0)), 'frac', round(r.get('frac',0),3), d.get('clocks'), 'e2e', d.get('e2e',{}).get('value'))
        elif 'rc=' in l or 'Error' in l: print(f, l.strip())
