#!/bin/bash
NO_BENCH=1 TEST_TIMEOUT=600 bash scripts/gpu_tests.sh
STEPS=30 bash scripts/bench_all.sh
VAR=SGWLS_KA_CTA_WARPS VALS="2 8" CONFIGS="c5 c3 c4" STEPS=30 bash scripts/ab_env.sh
