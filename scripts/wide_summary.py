"""Summarise the wide-grid A/B bench lines and ncu raw pages (gpurun_out/wide_<tag>_*)."""
import json,glob,sys,csv
tag=sys.argv[1]
for f in sorted(glob.glob(f'gpurun_out/wide_{tag}_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, 'ERR'); continue
    k=d['kernels']
    print(f.split('/')[-1][:-5].ljust(34), '%.3e'%d['value'], 'ms %.1f'%d['ms_per_step'], 'mhz', d['clocks']['sm_mhz'],
      ' '.join('%s %.2fms %.0f'%(n[:6], v['ms_total']/v['launches'], v['gbs']) for n,v in k.items()))
for f in sorted(glob.glob(f'gpurun_out/wide_{tag}_*_raw.csv')):
    rows=list(csv.reader(open(f))); hdr=rows[0]
    g=lambda r,w: r[hdr.index(w)]
    print(f)
    for r in rows[2:]:
        print('  ', g(r,'Kernel Name')[:40], g(r,'gpu__time_duration.sum'), 'rd', g(r,'dram__bytes_read.sum'), 'wr', g(r,'dram__bytes_write.sum'), 'hit', g(r,'lts__t_sector_hit_rate.pct')[:5])
for f in sorted(glob.glob(f'gpurun_out/wide_{tag}_*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception: continue
    if d.get('mg'):
        print(f.split('/')[-1][:-5].ljust(34), 'MG %.3f ms/cycle' % d['mg']['ms_per_iteration'],
              'PCG %.3f ms/it' % d['pcg']['ms_per_iteration'] if d.get('pcg') else '', 'frac', d['roofline']['frac'])
