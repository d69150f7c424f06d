#!/bin/bash
NOVA_DEC_FUSED_DBG=1 NOVA_DEC_FUSED_STOP=4 NOVA_DEC_FUSED_HALT=1 timeout 120 python tests/dbg_fused.py halt 2>&1 | grep -v Warn | tail -4
NOVA_DEC_FUSED_DBG=2 NOVA_DEC_FUSED_STOP=4 NOVA_DEC_FUSED_HALT=1 timeout 120 python tests/dbg_fused.py halt 2>&1 | grep -v Warn | tail -1 | cut -c1-400
