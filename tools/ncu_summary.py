"""Summarise ncu outputs into profiles/: launch list (per-kernel time share, DRAM bytes) and
key metrics of the --set full captures.  usage: ncu_summary.py launches.csv out.md [prof.ncu-rep ...]"""
import csv, subprocess, sys, collections
launch_csv, out = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(launch_csv)))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(',', ''))
    names[r[ii]] = r[ki].split('(')[0]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for lid, m in per.items():
    a = agg[names[lid]]
    a[0] += 1; a[1] += m.get('gpu__time_duration.sum', 0); a[2] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
lines = ["# ncu launch list summary (cold-cache, serialised replay: compare SHARES, not absolutes)", "",
         f"source: {launch_csv}; {len(per)} launches; total {tot/1e3:.1f} us", "",
         "| kernel | launches | total us | share | mean us | DRAM bytes/launch |", "|---|---|---|---|---|---|"]
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"| {k} | {a[0]} | {a[1]/1e3:.1f} | {100*a[1]/tot:.1f}% | {a[1]/a[0]/1e3:.2f} | {a[2]/a[0]:.3g} |")
for rep in sys.argv[3:]:
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) < 3:
        continue
    hdr, val = rr[0], rr[2]
    want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
            'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
            'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
            'smsp__inst_executed.sum', 'l1tex__t_bytes.sum', 'lts__t_bytes.sum']
    lines += ["", f"## {rep.split('/')[-1]}", "", "| metric | value |", "|---|---|"]
    for wname in want:
        for i, k in enumerate(hdr):
            if k == wname:
                lines.append(f"| {k} | {val[i]} |")
    # hottest stall reasons
    st = [(hdr[i], val[i]) for i in range(len(hdr)) if hdr[i].startswith('smsp__pcsamp_warps_issue_stalled_') and not hdr[i].endswith('not_issued')]
    st = sorted(((k, float(v.replace(',', ''))) for k, v in st if v.replace(',', '').replace('.', '').isdigit()), key=lambda x: -x[1])[:6]
    lines.append("| top stall reasons (samples) | " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(v)}" for k, v in st) + " |")
open(out, 'w').write("\n".join(lines) + "\n")
print("\n".join(lines))
