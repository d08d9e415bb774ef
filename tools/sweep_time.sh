#!/bin/bash
# cfg-2 matvec times per degree (median of 20), stored coefficients: tools/sweep_time.sh [degrees...]
cd "$(dirname "$0")/.."
for p in ${@:-2 3 4 5 6}; do python tools/profile_matvec.py --p $p --reps 20 2>&1 | grep matvec; done
