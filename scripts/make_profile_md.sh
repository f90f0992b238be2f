#!/bin/bash
# Turn the gpurun_out/prof_* captures of scripts/capture_profiles.sh into profiles/<round>_*.md.
cd "$(dirname "$0")/.."
S=scripts/summarize_ncu.py
R=${1:-r2}
{ echo "# ${R} — cfg3 TI-Sinkhorn (N=M=65536, d=2, fp32), \`python bench.py --no-secondary --steps 1 --warmup 3\` (a step = one 200-iteration solve)"; echo;
  echo "## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised — compare shares)"; echo;
  python $S launches gpurun_out/prof_cfg3_launches.csv; echo;
  echo "probe_ex2 is the MUFU peak microbenchmark bench.py runs live beside the fixed denominator (not part of a step)."; echo;
  echo "## Full capture of the dominant kernel (ncu --set full --clock-control none, -k regex:sk_main -s 40 -c 1)"; echo;
  python $S full gpurun_out/prof_cfg3_full.ncu-rep; echo;
  echo "Reading: XU (MUFU) pipe ~93% busy; DRAM traffic per launch is the row records and column data only (no re-reads). Bound = MUFU ex2 throughput."; } > profiles/${R}_cfg3_sinkhorn.md
cp gpurun_out/prof_cfg3_launches.csv profiles/${R}_cfg3_launches.csv
{ echo "# ${R} — cfg2 batched 1-D FW (B=296 slice of 4096, N=M=1024, fp64, 20 line-search iterations): \`python scripts/prof_fw.py 296 20 linesearch\`"; echo;
  echo "## Launch list (cold-cache, serialised — compare shares)"; echo; python $S launches gpurun_out/prof_fw_launches.csv; echo;
  echo "## Full capture of fw1d_kernel (ncu --set full --clock-control none)"; echo; python $S full gpurun_out/prof_fw_full.ncu-rep; echo;
  echo "### Instructions and stalls by source function (scripts/sass_regions.py, per warp-iteration = / (296 CTAs x 8 warps x 20 iterations))"; echo; echo '```';
  python scripts/sass_regions.py gpurun_out/prof_fw_full.ncu-rep paper_2201_00730_b200/build/fw1d.o fw1d_kernelILi4ELi0ELb0 paper_2201_00730_b200/csrc/fw1d_kernel.cuh $((296*8*20)) 2>/dev/null | head -45; echo '```'; } > profiles/${R}_cfg2_fw.md
{ echo "# ${R} — cfg5 barycenter FW (64 problems x K=16 x N=8192, fp64, 3 iterations): \`python scripts/prof_bary.py 64 3\`"; echo;
  echo "## Launch list (cold-cache, serialised — compare shares; mot_plan / mot_tilt / mot_lse / mot_finalize run once per solve)"; echo; python $S launches gpurun_out/prof_bary_launches.csv;
  for k in mot_update2 mot_bucket mot_split; do echo; echo "## Full capture: $k"; echo; python $S full gpurun_out/prof_bary_$k.ncu-rep; done; } > profiles/${R}_cfg5_barycenter.md
{ echo "# ${R} — cfg4 batched Sinkhorn d=64 on tcgen05 CTA pairs (64 of 256 problems, N=M=4096): \`python scripts/perf_cfg4.py 64\`"; echo;
  echo "## Launch list (cold-cache, serialised — compare shares)"; echo; python $S launches gpurun_out/prof_c4_launches.csv; echo;
  echo "## Full capture of sk_main_tc<64>"; echo; python $S full gpurun_out/prof_c4_full.ncu-rep; } > profiles/${R}_cfg4_tcgen05.md
cp gpurun_out/prof_c4_launches.csv profiles/${R}_cfg4_launches.csv
echo done
