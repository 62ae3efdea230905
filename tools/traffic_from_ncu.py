"""Per-phase DRAM bytes and kernel time per step from an ncu launch list of bench.py
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).
usage: traffic_from_ncu.py launches.csv WORKLOAD out.json"""
import collections, csv, json, sys
path, wl, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = collections.defaultdict(dict); names = {}
for r in rows[hi + 1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(',', ''))
    names[r[ii]] = r[ki].split('(')[0].replace('kkt::', '')
def phase(k):
    if k.startswith(('condense', 'dweights')): return 'condense'
    if k.startswith(('factor', 'linv', 'tile_factor', 'factor_block')): return 'factor'
    if k.startswith('at::') or 'elementwise' in k or 'Fill' in k: return None
    return 'solve'
def bare(k):
    return k.split('<')[0].replace('void ', '').strip()
steps = sum(1 for i in names if names[i] == 'condense_kernel')
byts = collections.Counter(); tns = collections.Counter()
kb = collections.Counter(); kt = collections.Counter(); kn = collections.Counter()
for i, m in per.items():
    p = phase(bare(names[i]))
    if p is None: continue
    b_ = m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
    byts[p] += b_
    tns[p] += m.get('gpu__time_duration.sum', 0)
    if bare(names[i]).startswith('tile_factor'):  # the large-supernode kernel
        byts['factor_large'] += b_
        tns['factor_large'] += m.get('gpu__time_duration.sum', 0)
    k = bare(names[i]); kb[k] += b_; kt[k] += m.get('gpu__time_duration.sum', 0); kn[k] += 1
res = {"workload": wl, "source": f"{path} ({steps} condense->factor->solve steps of bench.py under ncu, cold caches)",
       "steps": steps,
       "dram_bytes_per_step": {k: v / steps for k, v in byts.items()},
       "ncu_time_ns_per_step": {k: v / steps for k, v in tns.items()},
       "per_kernel": {k: {"launches_per_step": kn[k] / steps, "dram_bytes_per_step": kb[k] / steps,
                          "ncu_time_ns_per_step": kt[k] / steps} for k in kb}}
json.dump(res, open(out, 'w'), indent=1)
print(json.dumps(res))
