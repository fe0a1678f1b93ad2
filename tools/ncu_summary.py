"""Summarise ncu outputs into profiles/ (markdown).

  python tools/ncu_summary.py launches <launches.csv> <out.md>    # per-kernel share of the step
  python tools/ncu_summary.py full <report.ncu-rep> <out.md>      # one kernel, --set full
"""
import collections, csv, io, re, subprocess, sys


def short(n):
    n = re.sub(r'\(.*', '', n).replace('void ', '').replace('gemslr::', '')
    return n


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ik, iv = h.index('Kernel Name'), h.index('Metric Value')
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= iv:
            continue
        k = short(r[ik])
        tot[k] += float(r[iv].replace(',', ''))
        cnt[k] += 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total µs | µs/launch | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / 1e3 / cnt[k]:.2f} | {100 * v / T:.1f}% |")
    lines.append(f"\nTotal {T / 1e3:.1f} µs over {sum(cnt.values())} launches (ncu, `--clock-control none`, "
                 "serialised cold-cache launches: compare shares, not absolute times).")
    open(out, 'w').write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
           'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread', 'launch__grid_size',
           'launch__block_size', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'lts__t_bytes.sum',
           'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__inst_executed.sum']


def full(path, out):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = short(r[h.index('Kernel Name')])
        lines.append(f"### {name}\n\n| metric | value | unit |\n|---|---|---|")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"| {m} | {r[i]} | {units[i]} |")
        # stall reasons
        st = []
        for i, k in enumerate(h):
            if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
                try:
                    v = float(r[i].replace(',', ''))
                except ValueError:
                    continue
                if v > 0:
                    st.append((v, k.replace('smsp__pcsamp_warps_issue_stalled_', '')))
        st.sort(reverse=True)
        T = sum(v for v, _ in st) or 1
        lines.append("\nWarp stall samples: " + ", ".join(f"{k} {100 * v / T:.1f}%" for v, k in st[:8]) + "\n")
    open(out, 'w').write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == '__main__':
    {'launches': launches, 'full': full}[sys.argv[1]](sys.argv[2], sys.argv[3])
