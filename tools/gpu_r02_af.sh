#!/bin/bash
# conv (persistent grid capped at G CTAs) concurrent with the pair ReLU on another stream
for g in 148 120 100 80; do echo "grid=$g $(HB_TMA_GRID=$g timeout 300 python tools/diag_overlap.py 2>/dev/null)"; done
