#!/bin/bash
# One profiling pass of the current tree (run on the GPU box from the repo root):
#   tools/profile_round.sh TAG
# -> gpurun_out/bench_TAG.json          the default bench line (no profiler)
#    gpurun_out/launches_TAG.csv        ncu launch list of the same command
#    gpurun_out/tree_TAG.ncu-rep        ncu --set full of one tree_kernel launch
#    gpurun_out/ribbon_TAG.ncu-rep      ncu --set full of the first elim + forms launches
set -e
TAG=$1
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_TAG.tmp 2> gpurun_out/bench_$TAG.err
mv gpurun_out/bench_TAG.tmp gpurun_out/bench_$TAG.json
tail -1 gpurun_out/bench_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --leaf-configs "" --query-reps 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tree_kernel -s 2 -c 1 -o gpurun_out/tree_$TAG \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --leaf-configs "" --queries 0 > gpurun_out/ncu_tree_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"ribbon_(elim|forms)" -s 40 -c 2 -o gpurun_out/ribbon_$TAG \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --leaf-configs "" --queries 0 > gpurun_out/ncu_ribbon_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"bk_l1_scatter|bk_cluster_sort|ribbon_keyrows_bins" -s 6 -c 3 -o gpurun_out/bucket_$TAG \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --leaf-configs "" --queries 0 > gpurun_out/ncu_bucket_$TAG.log 2>&1
echo done
