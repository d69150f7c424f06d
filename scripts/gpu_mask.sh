#!/bin/bash
for M in 0 4 12 14 28 30 31; do
  for S in 0 24 40 80; do NOVA_DEC_TMA=$M timeout 120 python scripts/pass_profile.py --stage dec --B 2 --split $S 2>/dev/null | sed "s/^/{\"mask\": $M, /; s/{\"mask\": $M, {/{\"mask\": $M, /"; done
done
for M in 0 31 28; do NOVA_DEC_TMA=$M timeout 120 python scripts/pass_profile.py --stage dec --B 8 --split 0 2>/dev/null | sed "s/^{/{\"mask\": $M, /"; done
