"""Summarise an ncu --page source --print-source=sass CSV: hottest SASS instructions by
warp-stall samples, with a little context.  usage: ncu_hot.py file.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
tot = sum(float(d['Warp Stall Sampling (All Samples)'] or 0) for d in data)
idx = sorted(range(len(data)), key=lambda i: -float(data[i]['Warp Stall Sampling (All Samples)'] or 0))
for i in idx[:N]:
    d = data[i]
    s = float(d['Warp Stall Sampling (All Samples)'] or 0)
    prev = data[i - 1]['Source'].strip() if i else ''
    print('%5.1f%%  [%4d] %-50s  <- prev: %s' % (100 * s / tot, i, d['Source'].strip()[:50], prev[:45]))
print('total samples', tot)
