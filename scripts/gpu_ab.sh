#!/bin/bash
# parity of every schedule, then A/B of one knob on the bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -3
bash scripts/ab_env.sh
