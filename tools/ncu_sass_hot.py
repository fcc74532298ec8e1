"""Per-SASS-instruction stall breakdown of an ncu report (source page):
total samples by stall reason, and the hottest instructions with their reasons."""
import csv
import subprocess
import sys


def main(rep, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Address")
    idx = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {r: 0 for r in reasons}
    insts = []
    for r in rows:
        if len(r) != len(hdr) or not r[0].startswith("0x"):
            continue
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        per = {k: int(r[idx[k]] or 0) for k in reasons}
        for k, v in per.items():
            tot[k] += v
        insts.append((s, r[0][-5:], r[1].strip(), per))
    T = sum(tot.values()) or 1
    print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
    for s, a, src, per in sorted(insts, key=lambda x: -x[0])[:n]:
        top = ", ".join(f"{k[6:]} {v}" for k, v in sorted(per.items(), key=lambda x: -x[1])[:3] if v)
        print(f"{100 * s / T:5.2f}% {a} {src[:60]:60s} {top}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
