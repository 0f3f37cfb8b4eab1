# SASS evidence for the hot kernels (cuobjdump of the sm_100a build, no GPU needed):
#   bash profiles/sass_summary.sh > profiles/r02/sass_summary.md
O=build/obj/engine.o
echo "# SASS mnemonics of the hot kernels (cuobjdump -sass $O, sm_100a)"
echo
echo "| kernel | instructions | tensor / TMA / async evidence |"
echo "|---|---|---|"
python3 - "$O" <<'PY'
import subprocess, sys, re, collections
sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)[1:]
want = ["k_gemm_tma", "k_gemm_tc", "k_gemm_bulk", "k_aggregate_bulk", "k_aggregate<", "k_recompute_sparse", "k_expand_filter", "k_classify", "k_batch_group", "k_commit"]
keys = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "UTMAPF", "SYNCS", "LDGSTS", "FMUL", "FADD", "FFMA", "ATOMG", "RED"]
demangle = lambda n: subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
rows = {}
for f in funcs:
    name = demangle(f.split("\n", 1)[0].strip())
    short = re.sub(r"\(.*", "", name).replace("void ", "").replace("sgb::", "")
    if not any(w.replace("<", "") in short for w in want):
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,6}\*/\s+([A-Z0-9_.@!P ]+?)\s", f)
    mn = [re.sub(r"^@!?U?P\d+\s+", "", i).split(" ")[0] for i in ins]
    c = collections.Counter(m.split(".")[0] for m in mn)
    full = collections.Counter(m for m in mn if m.split(".")[0] in ("UTMALDG", "UTCHMMA", "UBLKCP", "LDTM"))
    ev = ", ".join(f"{k}x{c[k]}" for k in keys if c[k])
    det = ", ".join(f"{k}x{v}" for k, v in sorted(full.items()))
    rows.setdefault(short, (len(mn), ev + (f" [{det}]" if det else "")))
for k, (n, ev) in sorted(rows.items()):
    print(f"| `{k}` | {n} | {ev} |")
PY
