#!/bin/bash
# ncu evidence for the hot kernels (run on the GPU box via gpurun).
#   tools/profile.sh [tag] [kernels...]
# Writes gpurun_out/prof_<kernel>.ncu-rep (one --set full capture of one
# launch each) and gpurun_out/launches_<tag>.csv (the per-launch device-time
# list of one bench step, cold-cache and serialized: compare shares).
set -u
TAG=${1:-r01}
shift || true
WANT=${*:-"hotspot srad kmeans bfs needle lud ludp bpfwd bpadj gemm decide launches"}
OUT=gpurun_out
mkdir -p $OUT
unset GS_RING   # ncu serializes kernels: one decision launch per call (the default)
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  case " $WANT " in *" $name "*) ;; *) return ;; esac
  timeout 300 $NCU -k regex:$rx -s $skip -c 1 -o $OUT/prof_$name -f "$@" > $OUT/prof_$name.log 2>&1 \
    || echo "capture $name failed/timeout" >> $OUT/prof_errors.log
}
cap hotspot hotspot_pass4 1 python tools/debug_job.py hotspot 24576 16
cap srad srad_stream 3 python tools/debug_job.py srad 24576 5
cap kmeans kmeans_assign 2 python tools/debug_job.py kmeans 32000000 4 34
cap bfs bfs_expand 9 python tools/debug_job.py bfs 128000000
cap needle needle_bands 0 python tools/debug_job.py needle 24576
cap lud lud_internal 20 python tools/debug_job.py lud 6144
cap ludp lud_panel 20 python tools/debug_job.py lud 6144
cap bpfwd bp_forward 0 python tools/debug_job.py backprop 48000000 2 16
cap bpadj bp_adjust 1 python tools/debug_job.py backprop 48000000 2 16
cap gemm gemm_bf16_tc 4 python tools/debug_job.py yolo 608 1 32
cap decide gs_interp 0 python -c "import __graft_entry__ as g; g.smoke()"
case " $WANT " in *" launches "*)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $OUT/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --skip-e2e --skip-sa --skip-cfg2 --skip-cfg3 \
  --cpu-budget 1 > $OUT/launches_bench_$TAG.log 2>&1 || echo "launch list failed" >> $OUT/prof_errors.log ;;
esac
# per-capture DRAM traffic + duration summary (for profiles/)
for f in $OUT/prof_*.ncu-rep; do
  [ -e "$f" ] || continue
  ncu -i "$f" --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active > "${f%.ncu-rep}.csv" 2>/dev/null
done
