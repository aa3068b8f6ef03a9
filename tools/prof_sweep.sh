#!/bin/bash
for t in 2 3 4; do timeout 60 python tools/prof_kernel.py --t $t --reps 5; done 2>&1 | grep -v Warn
