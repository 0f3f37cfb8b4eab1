# One --set full capture of a profiled round (bench.py brackets its timed rounds with
# cudaProfilerStart/Stop under SGNN_BENCH_NCU_RANGE=1) and the warp-stall breakdown of
# every launch, plus the source-level counters of the kernels named in $SRC.
#   C=c2 V=v6 SRC="k_gemm_bulk k_recompute_sparse" bash profiles/ncu_stalls.sh
set -x
export SGNN_BENCH_NCU_RANGE=1
C=${C:-c2}
V=${V:-v6}
R=${R:-r02}
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --launch-skip 1 \
  --launch-count ${N:-40} -o /tmp/stall_${C}_${V} python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_stall_${C}.log 2>&1
python profiles/stall_summary.py /tmp/stall_${C}_${V}.ncu-rep > gpurun_out/${R}_${C}_stalls_${V}.md
python profiles/summarize_ncu.py /tmp/stall_${C}_${V}.ncu-rep gpurun_out/${R}_${C}_ncu_full_${V} > /dev/null
for k in ${SRC:-k_gemm_bulk}; do
  ncu -i /tmp/stall_${C}_${V}.ncu-rep --page source --csv -k regex:$k > gpurun_out/${R}_${C}_src_${k}_${V}.csv 2>&1
done
ls -la gpurun_out
