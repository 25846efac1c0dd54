"""Per-CUDA-source-line warp-stall samples from an ncu report (--import-source, -lineinfo):
`python tools/ncu_lines.py REPORT [N]`.  Sums the SASS rows under each source line of the
`--page source --print-source cuda,sass` export.  Diagnostic only."""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f, line, src = "?", None, ""
    acc = {}
    total = 0
    for r in csv.reader(txt.splitlines()):
        if len(r) == 2 and r[0] == "File Path":
            f = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) < 6 or r[0] == "Line No":
            continue
        if r[0]:
            line, src = r[0], r[1]
            continue
        try:
            s = int(r[4])
        except ValueError:
            continue
        total += s
        key = (f, line)
        a = acc.setdefault(key, [0, src.strip()[:100]])
        a[0] += s
    print("total samples", total)
    for (fn, ln), (s, sr) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{s:6d} {100.0 * s / max(total, 1):5.1f}%  {fn}:{ln}  {sr}")


if __name__ == "__main__":
    main()
