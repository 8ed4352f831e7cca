"""Top stalled SASS lines of one kernel in an ncu report.

    python tools/ncu_hot.py REPORT KERNEL_REGEX [LAUNCH_SKIP] [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, regex = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[0][1][:120])
    h = rows[1]
    ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    body = [x for x in rows[2:] if len(x) > ie]
    print("samples", sum(f(x[ws]) for x in body), "warp instructions", sum(f(x[ie]) for x in body))
    for x in sorted(body, key=lambda x: -f(x[ws]))[:top]:
        print(f"{int(f(x[ws])):6d} {int(f(x[ie])):8d}  {x[0][-6:]}  {x[1].strip()[:90]}")


if __name__ == "__main__":
    main()
