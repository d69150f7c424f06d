#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for M in 2b 7b; do for S in 0 32 64; do timeout 120 python scripts/pass_profile.py --model $M --stage dec --split $S 2>/dev/null; done; done
