"""Per-step kernel time breakdown from an ncu launch list (launches.csv)."""
import collections, csv, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]; data = rows[1:]
iN, iV, iU = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'ns': 1, 'nsecond': 1, 'us': 1e3, 'usecond': 1e3, 'ms': 1e6, 'msecond': 1e6}
names = [r[iN].split('(')[0].replace('void ', '') for r in data]
vals = [float(r[iV].replace(',', '')) * scale[r[iU]] for r in data]
first = [i for i, n in enumerate(names) if 'deim' in n][0]
tot, cnt = collections.Counter(), collections.Counter()
nsteps = sum(1 for n in names if 'deim' in n)
for n, v in zip(names[first:], vals[first:]):
    tot[n[:50]] += v; cnt[n[:50]] += 1
T = sum(tot.values())
print('steps', nsteps, 'kernel time per step (us)', round(T / nsteps / 1e3, 1))
for k, v in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{k:50s} {cnt[k]/nsteps:5.1f}/step {v/nsteps/1e3:8.1f} us/step {100*v/T:5.1f}%")
