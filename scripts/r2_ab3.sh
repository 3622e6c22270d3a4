#!/bin/bash
LIBS="default kbc2" CONFIGS="c4" STEPS=20 bash scripts/ab_lib.sh
VAR=SGWLS_KA_WARPS VALS="8" CONFIGS="c4" STEPS=20 bash scripts/ab_env.sh
VAR=SGWLS_TILE_WARPS VALS="8" CONFIGS="c4 c5" STEPS=20 bash scripts/ab_env.sh
