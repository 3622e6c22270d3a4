#!/bin/bash
CFG=c5 UNITS=111820800 LAUNCHES=1 bash scripts/ncu_r2.sh
