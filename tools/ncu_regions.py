"""Group an ncu source page (cuda,sass CSV) of the search kernel by code region.

    ncu -i REP --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_regions.py src.csv

Regions are located by marker comments in csrc/search.cu (the `// (a)` ...
`// (h)` step labels and the rerank/outputs headers), so the grouping follows
edits of the file.  Inlined helpers from search_common.cuh are grouped by
function.  Prints stall-sample, instruction and shared-wavefront shares.
"""
import collections
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2605_02171_b200", "csrc", "search.cu")
MARKERS = [  # (substring of the first line of a region, region name), in file order
    ("auto issue = [&]", "tma issue()"),
    ("if (a.qraw) {", "encode prologue"),
    ("// ---- per-query init", "init"),
    ("// (a) TMA-gather", "tma issue call"),
    ("// speculative prefetch", "spec adjacency"),
    ("// (b) SM2 distances", "emit"),
    ("// (a paired pass", "distance loop"),
    ("// (c) contender ranks", "ranks"),
    ("// (d) in-place merge", "merge"),
    ("// (e) tie stack", "tie"),
    ("// (f) pick", "pick"),
    ("// (g) adjacency row", "adjacency load"),
    ("// (h) visited filter", "visited+compact"),
    ("// ---- outputs", "outputs"),
    ("if (a.do_rerank) {", "rerank"),
    ("// rank by (score desc", "rank out"),
    ("// one thread per pair", "end"),
]
HDR = os.path.join(ROOT, "paper_2605_02171_b200", "csrc", "search_common.cuh")
COMMON = [("void csa(", "distance (Sm2Acc)"), ("uint32_t row_sm2(", "distance (row_sm2)"),
          ("uint32_t lower_bound_key(", "lower_bound_key"),
          ("uint32_t upper_bound_u32(", "upper_bound_u32"), ("group_stride(", "common (other)")]


def common_regions():
    lines = open(HDR).read().splitlines()
    out = []
    for text, name in COMMON:
        for i, l in enumerate(lines, 1):
            if text in l:
                out.append((i, name))
                break
    return sorted(out)


def regions():
    lines = open(SRC).read().splitlines()
    starts = []
    for text, name in MARKERS:
        for i, l in enumerate(lines, 1):
            if text in l and (not starts or i > starts[-1][0]):
                starts.append((i, name))
                break
    return starts


def main(path):
    rows = list(csv.reader(open(path)))
    blocks, cur, hdr = [], None, None
    for r in rows:
        if r and r[0] == "Line No":
            cur, hdr = [], r
            blocks.append(cur)
            continue
        if cur is not None and len(r) == len(hdr) and r[2] == "-":
            d = dict(zip(hdr[4:], r[4:]))
            try:
                cur.append((int(r[0]), r[1], int(d["Warp Stall Sampling (All Samples)"]),
                            int(d["Instructions Executed"]), int(d["L1 Wavefronts Shared"] or 0)))
            except ValueError:
                pass
    big = max(blocks, key=len)
    starts = regions()
    cstarts = common_regions()
    agg = collections.defaultdict(lambda: [0, 0, 0])
    tot = [0, 0, 0]
    for b in blocks:
        common = any("Harley" in x[1] or "csa(" in x[1] for x in b)
        for ln, src, smp, ins, wf in b:
            key = "other"
            if b is big:
                for st, name in starts:
                    if ln >= st:
                        key = name
            elif common:
                key = "common (other)"
                for st, name in cstarts:
                    if ln >= st:
                        key = name
            for i, v in enumerate((smp, ins, wf)):
                agg[key][i] += v
                tot[i] += v
    print(f"{'stall smp':>9s} {'instr':>7s} {'smem wf':>8s}  region")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{100 * v[0] / tot[0]:8.1f}% {100 * v[1] / tot[1]:6.1f}% {100 * v[2] / max(tot[2], 1):7.1f}%  {k}")
    print(f"totals: {tot[0]} samples, {tot[1]} warp-instructions, {tot[2]} shared wavefronts")


if __name__ == "__main__":
    main(sys.argv[1])
