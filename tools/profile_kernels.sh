#!/bin/bash
# ncu --set full of one launch of each main kernel of a steady config-4 sweep
# (tools/steady_sweep.py, sweep 3 inside cudaProfilerStart/Stop); text summaries by
# tools/ncu_sum.py.   usage (GPU box): bash tools/profile_kernels.sh <out_dir>
out=${1:-gpurun_out/kern}
mkdir -p "$out"
python tools/steady_sweep.py > "$out/plain.json" || exit 1
while read -r name regex skip; do
  ncu --profile-from-start off --clock-control none --set full --import-source on \
      -k "regex:$regex" -s "$skip" -c 1 -f -o "$out/$name" python tools/steady_sweep.py > "$out/$name.json" 2> "$out/$name.err"
  python tools/ncu_sum.py "$out/$name.ncu-rep" > "$out/$name.txt" 2>&1
  ncu -i "$out/$name.ncu-rep" --page details > "$out/$name.details.txt" 2>&1
  [ -n "$KEEP_REP" ] || rm -f "$out/$name.ncu-rep"  # gpurun_out merges at most 64 MiB
done <<'L'
gather_bits knn_gather_bits_kernel 0
gather256 knn_gather_kernel 1
gather_warp knn_gather_warp_kernel 1
merge_cta knn_merge_kernel 0
merge_warp knn_merge_warp_kernel 1
tc_screen tc_screen_kernel 0
update update_kernel 0
k2 ising_refine_cta_kernel 3
select trikey_select_kernel 0
snapshot snapshot_ising_kernel 0
resolve resolve_rows_kernel 0
dedup pair_dedup_kernel 0
L
