#!/bin/bash
NO_BENCH=1 TEST_TIMEOUT=600 bash scripts/gpu_tests.sh
LIBS="default kbm3 lazy1" CONFIGS="c5 c4 c3 c2 c1" STEPS=30 bash scripts/ab_lib.sh
VAR=SGWLS_K2_NG VALS="16 32" CONFIGS="c5 c4" STEPS=30 bash scripts/ab_env.sh
CFG=c5 UNITS=111837184 LAUNCHES=1 bash scripts/ncu_r2.sh
