#!/bin/bash
# Launch list of the bench's timed region + one `ncu --set full` capture of
# the top kernels (run under gpurun; outputs in gpurun_out/).
set -x
mkdir -p gpurun_out
TAG=${1:-prof}
GLOD_PROFILE_RANGE=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 4 --warmup 10 --no-cpu-baseline \
  > gpurun_out/${TAG}_launches.log 2>&1
python tools/launches.py gpurun_out/${TAG}_launches.csv 4 > gpurun_out/${TAG}_launches_summary.txt
GLOD_PROFILE_RANGE=1 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k "regex:${KERNELS:-blend_bwd|adam_records|blend_fwd|preprocess|compact_kernel|ssim_pass1|load_blocks|pack_blocks}" -c ${COUNT:-9} \
  -o gpurun_out/${TAG}_full -f python bench.py --steps 2 --warmup 10 --no-cpu-baseline \
  > gpurun_out/${TAG}_full.log 2>&1
ls -la gpurun_out
