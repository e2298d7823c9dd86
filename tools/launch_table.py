"""Print per-launch times (and DRAM bytes when present) from an ncu --csv launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = {}
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if 'b200' not in d['Kernel Name']: continue
        data.setdefault(d['ID'], {'name': d['Kernel Name']})[d['Metric Name']] = float(d['Metric Value'])
tot = 0
for i, d in data.items():
    t = d['gpu__time_duration.sum'] / 1e3; tot += t
    extra = ''
    if 'dram__bytes_read.sum' in d:
        rb, wb = d['dram__bytes_read.sum'], d['dram__bytes_write.sum']
        extra = ' %.0f GB/s' % ((rb + wb) / (t * 1e-6) / 1e9)
    print('%-58s %9.1f us%s' % (d['name'].replace('void b200::', '')[:58], t, extra))
print('total %.1f us' % tot)
