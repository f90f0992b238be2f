#!/bin/bash
# Round-end ncu evidence (run on the GPU box under gpurun; each command first
# runs once without ncu).  Outputs go to gpurun_out/prof_*; then run
# scripts/make_profile_md.sh here to refresh profiles/*.md.  gpurun brings back
# at most 64 MiB, so the captures come in parts: capture_profiles.sh {1,2,3}.
set -x
O=gpurun_out
part=${1:-all}
if [ "$part" = 1 ] || [ "$part" = all ]; then
# cfg3 headline: launch list of a short bench run + full capture of the main kernel
# (a step is a whole 200-iteration solve: 1 timed + 3 warm-up solves and the e2e leg's 3)
timeout 300 python bench.py --no-secondary --steps 1 --warmup 3 > /dev/null && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/prof_cfg3_launches.csv python bench.py --no-secondary --steps 1 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sk_main -s 40 -c 1 -f -o $O/prof_cfg3_full python bench.py --no-secondary --steps 1 --warmup 3 > /dev/null 2>&1
# cfg2 FW: 296 problems x 20 iterations
timeout 300 python scripts/prof_fw.py 296 20 linesearch && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/prof_fw_launches.csv python scripts/prof_fw.py 296 20 linesearch > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fw1d_kernel -c 1 -f -o $O/prof_fw_full python scripts/prof_fw.py 296 20 linesearch > /dev/null 2>&1
fi
if [ "$part" = 2 ] || [ "$part" = all ]; then
# cfg5 barycenter: all 64 problems, 3 iterations
timeout 300 python scripts/prof_bary.py 64 3 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/prof_bary_launches.csv python scripts/prof_bary.py 64 3 > /dev/null 2>&1
for k in mot_update2 mot_bucket mot_split; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f -o $O/prof_bary_$k python scripts/prof_bary.py 64 3 > /dev/null 2>&1
done
fi
if [ "$part" = 3 ] || [ "$part" = all ]; then
# cfg4: 64 of the 256 problems
timeout 300 python scripts/perf_cfg4.py 64 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/prof_c4_launches.csv python scripts/perf_cfg4.py 64 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sk_main_tc -s 2 -c 1 -f -o $O/prof_c4_full python scripts/perf_cfg4.py 64 > /dev/null 2>&1
fi
ls -la $O
