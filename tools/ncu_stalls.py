"""Top stalled SASS instructions per kernel of an ncu report (source page, -lineinfo):
python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(path, top=16):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif r and r[0] == "Address" and cur is not None:
            cur[1] = r
        elif cur is not None and cur[1] is not None:
            cur[2].append(r)
    for name, h, rs in blocks:
        si = h.index("Warp Stall Sampling (All Samples)")
        tot = sum(int(x[si] or 0) for x in rs)
        print("=====", name[:90], "samples", tot)
        for x in sorted(rs, key=lambda x: -int(x[si] or 0))[:top]:
            d = dict(zip(h, x))
            st = {k[6:]: d[k] for k in h if k.startswith("stall_") and "(" not in k and d[k] not in ("0", "")}
            print(f"{d[h[si]]:>6} {d['Address'][-5:]} {d['Source'][:58]:58} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 16)
