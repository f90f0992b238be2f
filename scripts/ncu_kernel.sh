#!/bin/bash
# full ncu capture of one kernel of a short cfg5 run: ncu_kernel.sh <regex> <tag> [script args...]
re=$1; tag=$2; shift 2
ncu --set full --import-source on --clock-control none -k regex:$re -c 1 -f -o gpurun_out/$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
echo done
