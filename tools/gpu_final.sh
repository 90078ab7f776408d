#!/bin/bash
# round measurement + sanitizer runs of the final kernels
bash tools/gpu_round2.sh
bash tools/gpu_san2.sh
exit 0
