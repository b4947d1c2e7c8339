#!/bin/bash
# ncu --set full captures of the lane kernel: C=8 (no decisions), C=1 (forced victims), C=6 (heaviest),
# and config 3's latency-mode C=3 launch.  Usage: bash tools/gpu_prof_r2.sh TAG
TAG=${1:-r2}
for C in 8 1 6; do bash tools/gpu_ncu.sh ${TAG}_C$C "replay_lane_kernel<.int.$C," --parity-sample 0; done
bash tools/gpu_ncu.sh ${TAG}_cfg3 "replay_lane_kernel<.int.3," --config 3 --parity-sample 0
