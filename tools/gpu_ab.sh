#!/bin/bash
# A/B of the variants built by `python tools/ab_variants.py build` (interleaved rounds), on one
# GPU: tools/gpu_ab.sh <tag> <mode>... with modes of tools/ab_variants.py run (bench, fused, fwd,
# bwd, fused32, fwd32, bwd32, flow [FLOW_ARGS], batcher, scatter); "base:<mode>" adds a
# --clock-control base ncu timing of every variant for prof_fused <mode>.
set -u
mkdir -p gpurun_out
O=gpurun_out/$1; shift
for m in "$@"; do
  case $m in
    base:*)
      for so in paper_2602_05765_b200/variants/*.so; do
        echo "== $(basename $so .so) ${m#base:}" >> ${O}_base.log
        RLVLA_LIB=$so timeout -s KILL 600 ncu --clock-control base --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:lp_ -s 1 -c 1 --csv python tools/prof_fused.py --mode ${m#base:} --iters 1 2>&1 | grep -E '^"[0-9]' >> ${O}_base.log
      done ;;
    *)
      echo "== $m" >> ${O}_ab.log
      timeout -s KILL 1500 python tools/ab_variants.py run $m >> ${O}_ab.log 2>&1; echo "rc=$?" >> ${O}_ab.log ;;
  esac
done
echo done
