"""Summarise pers_timeline.py output: mean split duration per operand stage,
stage period and MMA-warp wait on op_full over stages 11-41, per variant block
(lines '== variant NAME' separate the blocks)."""
import re, sys
cur, data = None, {}
for line in open(sys.argv[1]):
    if line.startswith("== variant"):
        cur = line.split(None, 2)[2].strip()
        data[cur] = []
    m = re.match(r"stage\s+(\d+) split: wait_stg\s+(-?\d+) stg_ok\s+(-?\d+) opslot_ok\s+(-?\d+) "
                 r"done\s+(-?\d+) \| mma: wait\s+(-?\d+) go\s+(-?\d+)", line)
    if m and cur is not None and 11 <= int(m.group(1)) <= 41:
        data[cur].append([int(x) for x in m.groups()])
for k, v in data.items():
    if len(v) < 5:
        print(k, "no data")
        continue
    split = sum(r[4] - r[3] for r in v) / len(v)
    period = (v[-1][4] - v[0][4]) / (len(v) - 1)
    wait = sum(r[6] - r[5] for r in v) / len(v)
    print(f"{k:24s} split {split:6.0f} ns  period {period:6.0f} ns  mma wait {wait:5.0f} ns")
