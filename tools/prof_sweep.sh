#!/bin/bash
for t in 2 3 4; do timeout 60 python tools/prof_kernel.py --t $t --reps 5; done 2>&1 | grep -v Warn
timeout 60 python tools/prof_kernel.py --t 4 --n 1024 --reps 3 2>&1 | grep -v Warn
