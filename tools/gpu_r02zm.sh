#!/bin/bash
# sustained (4 s, power-capped) A/B of the fused bidirectional sweep: single-block (k6_bidir_2a 0) against the CTA pair (2)
mkdir -p gpurun_out
{ for i in 1 2; do
    echo "== single-block (k6_bidir_2a=0)"; K6_CLOCK_BIDIR=1 PROHD_OPT_K6_BIDIR_2A=0 timeout 300 python tools/time_k6_clock.py 256 128
    echo "== pair (k6_bidir_2a=2)"; K6_CLOCK_BIDIR=1 PROHD_OPT_K6_BIDIR_2A=2 timeout 300 python tools/time_k6_clock.py 256 128
  done; } > gpurun_out/m_ab.txt 2>&1
