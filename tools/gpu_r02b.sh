#!/bin/bash
timeout 600 python tools/split_probe.py > gpurun_out/r02b_probe.log 2>&1
