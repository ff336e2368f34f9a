#!/bin/bash
# ncu evidence for the hot kernels (run on the GPU box via gpurun).
#   tools/profile.sh [tag]
# Writes gpurun_out/prof_<kernel>.ncu-rep and gpurun_out/launches_<tag>.csv.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
export GS_NO_RING=1   # ncu serializes kernels: use one decision launch per call
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 240 $NCU -k regex:$rx -s $skip -c 1 -o $OUT/prof_$name -f "$@" > $OUT/prof_$name.log 2>&1 \
    || echo "capture $name failed/timeout" >> $OUT/prof_errors.log
}
cap hotspot hotspot_step 5 python tools/debug_job.py hotspot 8192 10
cap srad srad_update 3 python tools/debug_job.py srad 8192 5
cap kmeans kmeans_assign 2 python tools/debug_job.py kmeans 4000000 4 34
cap bfs bfs_expand 5 python tools/debug_job.py bfs 16000000
cap needle needle_diag 300 python tools/debug_job.py needle 8192
cap lud lud_internal 20 python tools/debug_job.py lud 4096
cap bpfwd bp_forward 1 python tools/debug_job.py backprop 16000000 2 16
cap bpadj bp_adjust 1 python tools/debug_job.py backprop 16000000 2 16
cap decide gs_interp 0 python -c "import __graft_entry__ as g; g.smoke()"
# launch list of one (small) bench step: per-launch device time, cold-cache, serialized
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --jobs 8 --skip-e2e --skip-sa \
  --cpu-budget 1 > $OUT/launches_bench_$TAG.log 2>&1 || echo "launch list failed" >> $OUT/prof_errors.log
