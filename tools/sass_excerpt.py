"""profiles/<round>/f_sass_sweeps.txt: SASS excerpts of the two sweeps (bulk-copy tile fill, stretch inner loops) from the built library.
    python tools/sass_excerpt.py > profiles/r2/f_sass_sweeps.txt"""
import re
import subprocess
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_2603_05493_b200" / "libks_b200.so"
X = "_ZN3ksb12k_sweep_x_dcILi3ELb0ELi1EEEvNS_8EsdfViewENS_8TsdfViewEij"
Y = "_ZN3ksb12k_sweep_y_dcILi2ELi1EEEvNS_8EsdfViewEijj"


def sass(fun):
    text = subprocess.run(["cuobjdump", "-sass", "-fun", fun, str(LIB)], capture_output=True, text=True).stdout
    out = []
    for line in text.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if m:
            out.append(f"  /*{m.group(1)}*/ {m.group(2).strip()} ;")
    return out


def main():
    print("SASS excerpts of the two sweeps at HEAD (cuobjdump -sass of libks_b200.so, sm_100a; instruction text only, encodings dropped).\n"
          "What to look for: UBLKCP (cp.async.bulk global->shared, issued by one thread), SYNCS.* (mbarrier arrive.expect_tx / try_wait),\n"
          "CREDUX.MAX (redux.sync.max: the warp-wide longest window), VIADDMNMX.U32 (add + unsigned min in ONE instruction: a candidate's\n"
          "key for one position of a stretch), VIMNMX3 (three-way min of the top-level scans).\n")
    for title, fun, pats in [("k_sweep_x_dc<3,false,1> (cfg2 / cfg5env x sweep): tile fill by bulk copy + mbarrier", X, ["UBLKCP", "SYNCS"]),
                             ("k_sweep_x_dc<3,false,1>: stretch inner loop (7 running minima per candidate: IMAD + VIADDMNMX each)", X, None),
                             ("k_sweep_y_dc<2,1>: stretch inner loop", Y, None)]:
        lines = sass(fun)
        print("== " + title)
        if pats:
            keep = set()
            for i, l in enumerate(lines):
                if any(p in l for p in pats):
                    keep.update(range(max(0, i - 3), min(len(lines), i + 4)))
            prev = None
            for i in sorted(keep):
                if prev is not None and i != prev + 1:
                    print("  ...")
                print(lines[i])
                prev = i
        else:
            idx = [i for i, l in enumerate(lines) if "VIADDMNMX" in l]
            start = next(s for s in idx if len([j for j in idx if s <= j < s + 40]) >= 7)
            end = start
            while end < len(lines) and "BRA" not in lines[end]:
                end += 1
            print("\n".join(lines[max(0, start - 12):end + 1]))
        counts = {}
        for l in lines:
            for p in ["VIADDMNMX", "VIMNMX3", "VIMNMX", "CREDUX", "UBLKCP", "SYNCS", "LDS", "LDG", "STG", "ATOMS", "BAR.SYNC", "IMAD", "MUFU"]:
                if re.search(r"\b" + p + r"\b|\b" + p + r"\.", l):
                    counts[p] = counts.get(p, 0) + 1
        print("  static instruction counts: " + ", ".join(f"{k} {v}" for k, v in sorted(counts.items())) + f"; total {len(lines)}\n")


if __name__ == "__main__":
    main()
