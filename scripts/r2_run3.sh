#!/bin/bash
NO_BENCH=1 TEST_TIMEOUT=600 bash scripts/gpu_tests.sh
STEPS=30 bash scripts/bench_all.sh
CFG=c5 UNITS=111820800 bash scripts/ncu_r2.sh
