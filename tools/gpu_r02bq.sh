#!/bin/bash
# Round 2bq: ncu traffic capture and round-end rehearsal on the final sources
bash tools/gpu_ncu_summary.sh
bash tools/gpu_roundend.sh
