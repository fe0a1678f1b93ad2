"""Summarise ncu outputs into profiles/ (markdown).

  python tools/ncu_summary.py launches <launches.csv> <out.md>    # per-kernel share of the step
  python tools/ncu_summary.py full <report.ncu-rep> <out.md>      # one kernel, --set full
"""
import collections, csv, io, re, subprocess, sys


def short(n):
    n = re.sub(r'\(.*', '', n).replace('void ', '').replace('gemslr::', '')
    return n


def launches(path, out):
    """Per-kernel share of the NVTX-filtered solve launches, with DRAM bytes per
    launch when captured.  k_tri_reg launches come 7 per preconditioner apply
    (down l0, l1, l2, last, up l2, l1, l0); their classes are written to
    <out>.traffic.json for bench.py's roofline `traffic`."""
    import json
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ik, iv, iid = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID')
    imn = h.index('Metric Name') if 'Metric Name' in h else None
    per = collections.OrderedDict()          # launch id -> (kernel, {metric: value})
    for r in data:
        if len(r) <= iv:
            continue
        lid = int(r[iid])
        k = short(r[ik])
        m = r[imn] if imn is not None else 'gpu__time_duration.sum'
        per.setdefault(lid, (k, {}))[1][m] = float(r[iv].replace(',', ''))
    # Iterations queued after the done flag run as no-ops (every kernel exits at
    # once; the host reads the flag 6 iterations late): an iteration ends with
    # its k_fgmres_scale (CGS2) or k_dgs_upd (DCGS2), which moves >= 2 vectors when real; drop whole no-op
    # iterations so shares and per-launch figures describe real work.
    items = list(per.items())
    keep, seg = [], []
    for lid, (k, m) in items:
        seg.append((lid, (k, m)))
        if k.startswith('k_fgmres_scale') or k.startswith('k_dgs_upd'):
            b = m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
            if b >= 1e6 or 'dram__bytes_read.sum' not in m:
                keep.extend(seg)
            seg = []
    keep.extend(seg)
    dropped = len(items) - len(keep)
    tot, cnt, dram = collections.defaultdict(float), collections.Counter(), collections.defaultdict(float)
    tri = []
    for lid, (k, m) in keep:
        t = m.get('gpu__time_duration.sum', 0.0)
        unit_ns = 1.0
        tot[k] += t * unit_ns
        cnt[k] += 1
        b = m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
        dram[k] += b
        if k.startswith('k_tri_reg') or k.startswith('k_tri_pipe'):
            tri.append((t, b))
    T = sum(tot.values())
    lines = ["| kernel | launches | total µs | µs/launch | share | DRAM MB/launch |", "|---|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / 1e3 / cnt[k]:.2f} | {100 * v / T:.1f}% | {dram[k] / cnt[k] / 1e6:.2f} |")
    lines.append(f"\nTotal {T / 1e3:.1f} µs over {sum(cnt.values())} launches (ncu, `--clock-control none`, "
                 "serialised cold-cache launches: compare shares, not absolute times; "
                 f"{dropped} launches of iterations queued after the done flag, which exit at once, left out).")
    cls = {}
    if tri and len(tri) % 7 == 0:
        names = ['down_l0', 'down_l1', 'down_l2', 'last', 'up_l2', 'up_l1', 'up_l0']
        import statistics
        for i, nm in enumerate(names):
            sel = tri[i::7]
            cls[nm] = (statistics.median(t for t, _ in sel), statistics.median(b for _, b in sel))
        lines.append("\nTriangular-solve launches by position in the apply (median per launch):\n")
        lines.append("| launch | µs | DRAM MB |\n|---|---|---|")
        for nm, (t, b) in cls.items():
            lines.append(f"| {nm} | {t / 1e3:.1f} | {b / 1e6:.1f} |")
        def group(ks):
            return sum(cls[x][1] for x in ks) / len(ks)
        json.dump({"trisolve_down": group(['down_l0', 'down_l1', 'down_l2']),
                   "trisolve_up": group(['up_l0', 'up_l1', 'up_l2']), "trisolve_last": cls['last'][1],
                   "source": path}, open(out + '.traffic.json', 'w'), indent=1)
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
