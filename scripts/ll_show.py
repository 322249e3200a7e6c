"""Print the last call's kernels of an ncu launch-list CSV: python scripts/ll_show.py FILE"""
import csv, sys
rows = []
lines = [l for l in open(sys.argv[1]) if not l.startswith('==')]
for row in csv.DictReader(lines):
    rows.append((int(row['ID']), row['Kernel Name'], row['Grid Size'], row['Block Size'], float(row['Metric Value'].replace(',', ''))))
idx = [i for i, x in enumerate(rows) if 'range_kernel' in x[1]]
tot = 0
for x in rows[idx[-1]:]:
    print('  ', x[0], x[1][:64], x[2], x[3], x[4])
    tot += x[4]
print('sum', tot)
