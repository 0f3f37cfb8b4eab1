# A/B of library builds / engine switches on one box, alternating, 2 passes. A variant is
# name:ENV=VAL; another build is selected with SGNN_B200_LIB (the baseline build is made
# from a worktree of the baseline commit and copied to ablib/ before the gpurun call):
#   TAG=k1pre CONFIGS="c2 c3" VARIANTS="head:SGNN_B200_LIB=ablib/libstreamgnn_head.so new:X=1 nok1:SGNN_B200_K1PRE=0" bash profiles/ab_run.sh
mkdir -p gpurun_out/ab
for pass in 1 2; do
  for c in ${CONFIGS:-c2 c3}; do
    for v in $VARIANTS; do
      name=${v%%:*}; envs=${v#*:}
      env $envs timeout 600 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-e2e \
        > gpurun_out/ab/${TAG}_${c}_${pass}_${name}.json 2> gpurun_out/ab/${TAG}_${c}_${pass}_${name}.err
      python - gpurun_out/ab/${TAG}_${c}_${pass}_${name}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k = d.get("kernel_ms_per_step", {})
    print(sys.argv[1].split("/")[-1], "p50 %.4f mean %.4f" % (d["p50_ms"], d["ms_per_step"]),
          " ".join("%s=%.1f" % (a, 1000 * b) for a, b in k.items()), d.get("parity", {}).get("verify_full_inference"))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
    done
  done
done
