"""Attribute an ncu SASS source page (csv) to CUDA source lines via nvdisasm -gi line info.
usage: sass_lines.py <ncu_sass.csv> <nvdisasm -gi output> [top]"""
import collections
import csv
import re
import sys


def parse_disasm(path):
    secs, cur, loc, fresh = {}, None, None, False
    for line in open(path):
        m = re.match(r"\s*\.text\.(\S+):$", line) or re.match(r"^\.text\.(\S+):", line)
        if m:
            cur = m.group(1); secs[cur] = []; loc = None; continue
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', line)
        if m:
            # a group of comment lines precedes an instruction: the first is the innermost frame
            if not fresh:
                f = m.group(1).split("/")[-1]
                inl = re.search(r'inlined at "([^"]+)", line (\d+)', m.group(3))
                loc = f"{f}:{m.group(2)}" + (f" <- {inl.group(1).split('/')[-1]}:{inl.group(2)}" if inl else "")
                fresh = True
            continue
        fresh = False
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            secs[cur].append((m.group(2).strip(), loc))
    return secs


def norm(s):
    return re.sub(r"\s+", " ", s.split("`")[0]).strip().split(" ")[0]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) > ie]
    secs = parse_disasm(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    seqs = {k: [norm(i) for i, _ in v] for k, v in secs.items()}
    out_inst, out_samp = collections.Counter(), collections.Counter()
    i = 0
    while i < len(body):
        # find the section whose instruction sequence matches body[i:]
        best, blen = None, 0
        for k, sq in seqs.items():
            n = len(sq)
            if n == 0 or i + n > len(body):
                continue
            if all(norm(body[i + j][1]) == sq[j] for j in range(min(n, 64))) and \
               all(norm(body[i + j][1]) == sq[j] for j in range(n)):
                if n > blen:
                    best, blen = k, n
        if best is None:
            i += 1
            continue
        for j in range(blen):
            r = body[i + j]
            loc = secs[best][j][1] or "?"
            out_inst[loc] += float(r[ie] or 0)
            out_samp[loc] += float(r[ss] or 0)
        i += blen
    ti, ts = sum(out_inst.values()), sum(out_samp.values())
    print(f"total inst {ti:.0f}, samples {ts:.0f}")
    for loc, v in out_samp.most_common(top):
        print(f"{100*v/ts:5.1f}% samp {100*out_inst[loc]/ti:5.1f}% inst  {loc}")


if __name__ == "__main__":
    main()
