"""Top stalled SASS lines of one kernel from `ncu --page source --csv
--print-source sass` output: python profiles/ncu_top_stalls.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
k = 0
while k < len(rows):
    if rows[k] and rows[k][0] == "Kernel Name":
        name = rows[k][1]
        hdr = rows[k + 1]
        isrc, iss = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        data, j = [], k + 2
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            r = rows[j]
            try:
                data.append((float(r[iss]), j - k - 2, r[isrc].strip(),
                             {h: float(r[hdr.index(h)] or 0) for h in reasons}))
            except (ValueError, IndexError):
                pass
            j += 1
        tot = sum(d[0] for d in data) or 1
        print(f"== {name}  samples {tot:.0f}")
        for v, i, src, rs in sorted(data, reverse=True)[:n]:
            top = max(rs, key=rs.get)
            print(f"{v / tot:6.2%} #{i:5d} {top[6:]:>12} {src[:80]}")
        k = j
    else:
        k += 1
