#!/bin/bash
# round measurement (compute-sanitizer is closed on the GPU pool since r02q; tools/gpu_san2.sh
# still runs the sanitizer pass where it is available)
bash tools/gpu_round2.sh
exit 0
