"""Aggregate a compute-sanitizer log: counts of each reported error kind by the (device) source
locations involved, so a million identical hazards read as one line.

    python tools/sanitize_summary.py gpurun_out/sanitize/racecheck.log"""
import collections
import re
import sys


def main(path):
    kinds = collections.Counter()
    cur = None
    locs = []
    summary = []
    for ln in open(path, errors="replace"):
        ln = ln.rstrip("\n")
        if "SUMMARY" in ln or "sanitize cases ok" in ln:
            summary.append(ln.strip("= "))
        m = re.match(r"=+ (Error: .*?|Invalid .*?|Barrier error .*?|Leaked \d+ bytes|"
                     r"Warning: .*?)( at | in |\.|$)", ln)
        if m:
            if cur:
                kinds[(cur, tuple(locs[:2]))] += 1
            cur = re.sub(r"0x[0-9a-f]+", "*", m.group(1))
            locs = []
            continue
        m = re.search(r"(?:at|in) .*? in ([\w./]+\.(?:cu|cuh|cpp|h):\d+)", ln)
        if cur and m and "Host Frame" not in ln:
            locs.append(m.group(1))
    if cur:
        kinds[(cur, tuple(locs[:2]))] += 1
    print("\n".join(summary))
    for (k, loc), n in kinds.most_common(40):
        print("%8d  %s  @ %s" % (n, k, " / ".join(loc) or "-"))


if __name__ == "__main__":
    main(sys.argv[1])
