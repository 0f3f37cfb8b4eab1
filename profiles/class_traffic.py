"""Per-kernel-class DRAM traffic of one update round from a summarize_ncu.py json.

bench.py's roofline `traffic` for the dominant class (events / classify /
recompute) is the sum of dram__bytes_read + dram__bytes_write over that class's
launches in one round, read from profiles/ncu_<config>_summary.json.

    python profiles/class_traffic.py profiles/r01_c2_ncu_full_v6.json profiles/ncu_c2_summary.json
"""
import json
import sys

CLASSES = {
    "events": ("k_seed_records", "k_expand_records", "k_expand_filter", "k_self_records"),
    "classify": ("k_classify",),
    "recompute": ("k_aggregate", "k_recompute_sparse", "k_sparse_finalize"),
}
ROUND_START = ("k_batch_cluster", "k_batch_group_pre", "k_batch_group", "k_batch_keys")


def short(name):
    return name.replace("void ", "").split("(")[0].split("<")[0].split("::")[-1]


def main(src, out):
    recs = json.load(open(src))
    starts = [i for i, r in enumerate(recs) if short(r["kernel"]) in ROUND_START]
    a = starts[0] if starts else 0
    b = starts[1] if len(starts) > 1 else len(recs)
    rnd = [r for r in recs[a:b] if short(r["kernel"]) != "k_l2_flush"]
    res = {"source": f"{src} (ncu --set full, cold cache, one round: launches {a}..{b - 1})",
           "round_kernels": [r["kernel"].split("(")[0] for r in rnd]}
    for cls, names in CLASSES.items():
        mb = sum(r.get("dram_read_mb", 0) + r.get("dram_write_mb", 0) for r in rnd if short(r["kernel"]) in names)
        res[f"{cls}_dram_bytes_per_launch"] = mb * 1e6
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
