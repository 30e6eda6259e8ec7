"""Top CUDA source lines / SASS instructions by warp-stall samples in an ncu report
(ncu --page source --print-source cuda,sass; needs -lineinfo builds)."""
import csv, subprocess, sys


def hot(path, n=25, kernel=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["--kernel-name", "regex:" + kernel]
    raw = subprocess.run(cmd, capture_output=True, text=True).stdout
    fname, cur = "", ""
    by_line, by_inst, total = {}, [], 0.0
    for r in csv.reader(raw.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Line No", "Function Name"):
            continue
        if len(r) < 5:
            continue
        if r[0]:  # a CUDA source line
            cur = f"{fname}:{r[0]}  {r[1].strip()[:90]}"
            try:
                w = float(r[4] or 0)
            except ValueError:
                w = 0.0
            if r[2] == "" and w:
                by_line[cur] = by_line.get(cur, 0) + w
            continue
        if r[2].startswith("0x"):
            try:
                w = float(r[4] or 0)
            except ValueError:
                continue
            total += w
            by_inst.append((w, r[3].strip()[:55], cur))
            by_line.setdefault(cur + " [sass]", 0)
            by_line[cur + " [sass]"] += w
    tot = total or 1
    print("-- by source line (SASS samples attributed to the preceding source line)")
    for k, w in sorted(((k, w) for k, w in by_line.items() if k.endswith("[sass]")), key=lambda kv: -kv[1])[:n]:
        print(f"{100*w/tot:5.1f}%  {k[:-7]}")
    print("-- by instruction")
    for w, sass, src in sorted(by_inst, reverse=True)[:12]:
        print(f"{100*w/tot:5.1f}%  {sass:55s} | {src[:80]}")


if __name__ == "__main__":
    # ncu_hot_lines.py REPORT [KERNEL_REGEX ...]
    path, kernels = sys.argv[1], sys.argv[2:] or [None]
    for k in kernels:
        print("==", path, k or "")
        hot(path, n=12, kernel=k)
