# ncu launch list + one --set full round per config (run under gpurun from the repo root:
#   R=r02 V=v1 bash profiles/ncu_capture.sh). bench.py brackets its timed rounds with
# cudaProfilerStart/Stop when SGNN_BENCH_NCU_RANGE=1. The reports are summarised on the
# box (profiles/summarize_ncu.py, class_traffic.py) and left out of gpurun_out/ (size cap).
set -x
export SGNN_BENCH_NCU_RANGE=1
V=${V:-v6}
R=${R:-r02}
for c in ${CONFIGS:-c2 c3}; do
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_${c}_launches_${V}.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_list_${c}.log 2>&1
  python profiles/launch_summary.py gpurun_out/${R}_${c}_launches_${V}.csv 30 > gpurun_out/${R}_${c}_launches_${V}.txt
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --launch-skip 1 \
    --launch-count 32 -o /tmp/prof_${c}_${V} python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_full_${c}.log 2>&1
  python profiles/summarize_ncu.py /tmp/prof_${c}_${V}.ncu-rep gpurun_out/${R}_${c}_ncu_full_${V} > /dev/null
  python profiles/class_traffic.py gpurun_out/${R}_${c}_ncu_full_${V}.json gpurun_out/ncu_${c}_summary.json
  ncu -i /tmp/prof_${c}_${V}.ncu-rep --page source --csv -k regex:k_expand_filter > gpurun_out/${R}_${c}_filter_source_${V}.csv 2>&1
done
ls -la gpurun_out
