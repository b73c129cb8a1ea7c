"""Top source lines of an .ncu-rep by executed instructions and stall samples (needs -lineinfo builds).
    python tools/ncu_lines.py <rep> [top_n]"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur_file, hdr = None, None
    lines = {}
    for r in rows:
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0]:
            continue
        get = lambda name: r[hdr.index(name)]
        try:
            inst = int(get("Instructions Executed"))
            samp = int(get("# Samples"))
        except ValueError:
            continue
        if inst == 0 and samp == 0:
            continue
        key = (cur_file, int(r[0]))
        src = r[1].strip()
        old = lines.get(key, (0, 0, src))
        lines[key] = (old[0] + inst, old[1] + samp, src)
    tot_i = sum(v[0] for v in lines.values()) or 1
    tot_s = sum(v[1] for v in lines.values()) or 1
    print(f"total warp-instructions {tot_i}  stall samples {tot_s}")
    print("---- by instructions")
    for (f, ln), (i, s, src) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*i/tot_i:5.1f}% inst {100*s/tot_s:5.1f}% samp  {f}:{ln:<4d} {src[:110]}")
    print("---- by stall samples")
    for (f, ln), (i, s, src) in sorted(lines.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100*i/tot_i:5.1f}% inst {100*s/tot_s:5.1f}% samp  {f}:{ln:<4d} {src[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
