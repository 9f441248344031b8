"""Hot source lines from `ncu --page source --csv --print-source cuda,sass`:
warp-stall samples aggregated per (file, line)."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file, line_no, line_src = None, None, ""
    agg = defaultdict(float)
    src = {}
    total = 0.0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0]:  # a source line row
            line_no, line_src = r[0], r[1]
        if len(r) > 4 and r[2]:
            try:
                v = float(r[4])
            except ValueError:
                continue
            key = (cur_file, line_no)
            agg[key] += v
            src[key] = line_src
            total += v
    print(f"total stall samples {total:.0f}")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{v / total:6.1%} {key[0]}:{key[1]:>5}  {src[key].strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
