#!/bin/bash
# Round 2bo: final numbers (every config and name, ncu traffic capture) and the round-end rehearsal
bash tools/gpu_r02_final.sh r02bo
bash tools/gpu_roundend.sh
