#!/bin/bash
# tests, then A/B: weight laziness variants on every config, K2 tree widths on the small configs
NO_BENCH=1 TEST_TIMEOUT=600 bash scripts/gpu_tests.sh
LIBS="default kalazy lazy" CONFIGS="c5 c4 c3 c2 c1" STEPS=30 bash scripts/ab_lib.sh
VAR=SGWLS_K2_NG VALS="4 8 16 32" CONFIGS="c1 c2 c3 c5" STEPS=30 bash scripts/ab_env.sh
VAR=SGWLS_TILE_WARPS VALS="2 4 8" CONFIGS="c5 c4 c3" STEPS=30 bash scripts/ab_env.sh
VAR=SGWLS_KA_WARPS VALS="4 8" CONFIGS="c5 c3 c2" STEPS=30 bash scripts/ab_env.sh
