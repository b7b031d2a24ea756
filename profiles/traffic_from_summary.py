"""Per-task DRAM bytes of the roofline kernels from an ncu summary (profiles/<round>/
ncu_summary_*.md, written by scripts/final_evidence.sh) -> profiles/kernel_traffic.json.

    python profiles/traffic_from_summary.py profiles/r1h/ncu_summary_r1h.md r1h
"""
import json
import re
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
GROUPS = {"k_update": ["k_update"], "k_n0": ["k_n0"], "k_scale_tc": ["k_scale_tc"],
          "k_top": ["^k_top$", "k_live", "k_pairs"], "k_rsel": ["k_oexact", "k_rsel", "k_rsweep"],
          "k_select": ["k_rescore"]}


def main(path, tag):
    text = open(path).read()
    caps = {}
    for block in re.split(r"^#### capture ", text, flags=re.M)[1:]:
        head = block.splitlines()[0]
        m = re.match(r"(\S+) (\S+) \((\d+) tasks\)", head)
        if not m:
            continue
        k, cfg, n = m.group(1), m.group(2), int(m.group(3))
        tot = 0.0
        for what in ("dram read", "dram write"):
            mm = re.search(r"\| %s \| ([0-9.]+) (\w+) \|" % what, block)
            if mm:
                tot += float(mm.group(1)) * UNIT[mm.group(2)]
        caps[(k, cfg)] = tot / n
    out = {"note": "DRAM bytes (ncu dram__bytes_read.sum + dram__bytes_write.sum) per task of the "
                   "kernels behind each bench roofline stage, from the --set full captures in "
                   f"profiles/{tag}/ (one launch each); bench.py scales them to its own launch size. "
                   "k_update = k_update (k_terms is timed in the multi/injection stage), k_top = k_top + k_live + k_pairs, k_rsel = the winner report "
                   "(k_oexact + k_rsel + k_rsweep), k_select = k_rescore."}
    for cfg in sorted({c for _, c in caps}):
        out[cfg] = {g: sum(caps.get((k, cfg), 0.0) for k in ks) for g, ks in GROUPS.items()}
    json.dump(out, open("profiles/kernel_traffic.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
