#!/bin/bash
bash tools/c2_ab.sh "$1"
for lib in "" "$1"; do
RQ_LIB_PATH=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:reduce_tma -s 100 -c 2 python tools/overhead.py 2>&1 | grep -E "gpu__time" | tr -s ' ' | tr '\n' ' '; echo " ${lib:-tree}"
done
