#!/bin/bash
# barycenter parity tests + timing + launch list (gpurun helper)
tag=${1:-x}
python -m pytest tests/test_barycenter_gpu.py tests/test_scale_gpu.py tests/test_replay_gpu.py tests/test_cli_gpu.py -m gpu -q -x -k "bary or mot or cfg5 or barycenter" > gpurun_out/bary_tests_$tag.log 2>&1; echo rc=$? >> gpurun_out/bary_tests_$tag.log
python scripts/perf_bary.py > gpurun_out/perf_bary_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bary_launches_$tag.csv python scripts/prof_bary.py 64 3 > /dev/null 2>&1
echo done
