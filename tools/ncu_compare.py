"""Side-by-side raw ncu metrics of selected launches from several .ncu-rep
files: python tools/ncu_compare.py rep1:idx rep2:idx ... [--grep REGEX]"""
import csv
import re
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[2:]


def main():
    argv = sys.argv[1:]
    pat = None
    if "--grep" in argv:
        i = argv.index("--grep")
        pat = re.compile(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    args = argv
    cols = []
    for a in args:
        rep, idx = a.rsplit(":", 1)
        h, rows = load(rep)
        cols.append((a, dict(zip(h, rows[int(idx)]))))
    keys = [k for k in cols[0][1] if (pat is None or pat.search(k))]
    print("metric," + ",".join(c[0] for c in cols))
    for k in keys:
        print(k + "," + ",".join(c[1].get(k, "") for c in cols))


if __name__ == "__main__":
    main()
