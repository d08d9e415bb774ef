#!/bin/bash
# FD apply with and without programmatic dependent launch of the modal GEMMs (timing only)
cd "$(dirname "$0")/.."
for nopdl in 1 0; do
 for pn in "2,128" "4,128" "6,128" "4,256"; do
  IFS=, read p ne <<< "$pn"
  MFWQ_NO_PDL=$nopdl python tools/fd_time.py --p $p --n-el $ne | sed "s/^/no_pdl=$nopdl /"
 done
done
