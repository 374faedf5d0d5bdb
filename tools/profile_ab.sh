#!/bin/bash
# ncu summary of the engine kernel for two library builds (dev tool):
#   tools/profile_ab.sh WORKLOAD VARIANT... -> gpurun_out/ab_<variant>.ncu-rep
for v in "${@:2}"; do
  FBGPU_LIB=build/variants/$v/libfbgpu.so ncu --section SpeedOfLight --section WarpStateStats \
    --section InstructionStats --section LaunchStats --section Occupancy --clock-control none \
    -k regex:engine_kernel -c 1 -o gpurun_out/ab_$v -f python tools/ab_time.py $1 1 > /dev/null 2>&1
done
