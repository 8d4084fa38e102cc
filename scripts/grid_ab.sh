#!/bin/bash
# A/B of the generation loop's grid size (HGA_RUN_GRID caps the CTA count; results identical)
for g in 148 111 96 74 48; do
  echo "grid $g"
  HGA_RUN_GRID=$g timeout 300 python scripts/launch_cost.py 2>&1 | grep single | head -1
  HGA_RUN_GRID=$g timeout 300 python scripts/phase_timing.py 2>&1 | grep us_per_gen | head -4
done
