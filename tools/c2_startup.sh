bash tools/c2_iter.sh c2s
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:reduce_tma -s 100 -c 3 python tools/overhead.py 2>&1 | grep -E "gpu__time"
python tools/overhead.py 2>&1 | grep -v trace
