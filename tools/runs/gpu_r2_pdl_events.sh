#!/bin/bash
# does an event record between two PDL launches break the prologue overlap?
OUT=gpurun_out/${1:-pdl_events}
mkdir -p $OUT
for rep in 1 2; do
./build/cta_stamps dec 20 > $OUT/dec_noev_r$rep.json 2>&1
KG_STAMPS_EVENTS=1 ./build/cta_stamps dec 20 > $OUT/dec_ev_r$rep.json 2>&1
KG_PDL=0 ./build/cta_stamps dec 20 > $OUT/dec_nopdl_r$rep.json 2>&1
done
