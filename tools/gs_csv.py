"""Per-launch time / DRAM bytes of the Gram-Schmidt kernels in an ncu CSV (tools/gs_prof.py capture).

  python tools/gs_csv.py <capture.csv> [every]
"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
every = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ik, iv, iid, imn = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID'), h.index('Metric Name')
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    k = re.sub(r'\(.*', '', r[ik]).replace('void ', '').replace('gemslr::', '')
    per.setdefault(int(r[iid]), [k, {}])[1][r[imn]] = float(r[iv].replace(',', ''))
tot = collections.Counter()
for i, (k, m) in enumerate(per.values()):
    t = m['gpu__time_duration.sum'] / 1e3
    by = m['dram__bytes_read.sum'] + m['dram__bytes_write.sum']
    tot[k] += t
    if i % every == 0:
        print(f"{i:4d} {k[:36]:36s} {t:8.1f} us {by / 1e6:8.1f} MB {by / t / 1e3:7.0f} GB/s")
for k, t in tot.items():
    print(f"total {k:40s} {t:9.1f} us")
print(f"total {sum(tot.values()):.1f} us")
