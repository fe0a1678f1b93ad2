"""Print SASS of one kernel with the control bits decoded (stall, yield, write/read
scoreboard, wait mask) — to see which instructions wait on which scoreboards.
usage: python tools/sass_ctrl.py <binary> <kernel-name-substring> [start_addr end_addr]"""
import re, subprocess, sys

binary, name = sys.argv[1], sys.argv[2]
lo_a = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi_a = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 40
out = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout.splitlines()
on = False
prev = None
for ln in out:
    if "Function :" in ln:
        on = name in ln
        continue
    if not on:
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);\s*/\* 0x([0-9a-f]{16}) \*/", ln)
    if m:
        prev = (int(m.group(1), 16), m.group(2).strip())
        continue
    m = re.match(r"\s*/\* 0x([0-9a-f]{16}) \*/", ln)
    if m and prev:
        hi = int(m.group(1), 16)
        addr, ins = prev
        prev = None
        if not lo_a <= addr <= hi_a:
            continue
        stall, yld = (hi >> 41) & 0xF, (hi >> 45) & 1
        wr, rd, wm = (hi >> 46) & 7, (hi >> 49) & 7, (hi >> 52) & 0x3F
        tags = f"S{stall:02d}" + (" Y" if yld else "  ")
        tags += f" W{wr}" if wr != 7 else "   "
        tags += f" R{rd}" if rd != 7 else "   "
        tags += f" wait{{{','.join(str(b) for b in range(6) if wm >> b & 1)}}}" if wm else ""
        print(f"{addr:05x}  {tags:26s} {ins}")
