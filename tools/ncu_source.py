"""Top SASS lines of an .ncu-rep by executed instructions / stall samples (tooling)."""
import csv
import subprocess
import sys


def main(path, n=40, key="Instructions Executed"):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    i = next(k for k, ln in enumerate(lines) if ln.startswith('"Address"'))
    rows = list(csv.reader(lines[i:]))
    hdr = rows[0]
    ci, cs, cw = hdr.index(key), hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
    body = [r for r in rows[1:] if len(r) == len(hdr)]
    tot = sum(float(r[ci] or 0) for r in body)
    tots = sum(float(r[cw] or 0) for r in body)
    print(f"total {key}: {tot:.3e}  stall samples {tots:.0f}")
    for r in sorted(body, key=lambda r: -float(r[cw] or 0))[:n]:
        print(f"{float(r[ci] or 0):12.0f} {float(r[cw] or 0) / max(tots, 1):6.1%}  {r[cs].strip()[:90]}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
