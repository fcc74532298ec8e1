"""Summarise an ncu report's per-source-line warp stall samples (hottest lines)."""
import csv
import subprocess
import sys


def main(rep, n=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    path, agg, total = None, {}, 0.0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if len(r) > 4 and r[0].isdigit():
            try:
                v = float(r[4])
            except ValueError:
                continue
            key = (path, int(r[0]), r[1][:100])
            agg[key] = agg.get(key, 0.0) + v
            total += v
    for (p, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
        print(f"{100 * v / max(total, 1):5.1f}%  {p}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
