# A/B of the K12 row-kernel grid (CTAs per SM, RQ_XG_BPS) per workload
bash tools/ab_env.sh q6 "RQ_XG_BPS=0" "RQ_XG_BPS=8"; cp gpurun_out/ab_env.txt gpurun_out/ab_bps2_q6.txt
bash tools/ab_env.sh c3 "RQ_XG_BPS=0" "RQ_XG_BPS=3" "RQ_XG_BPS=6" "RQ_XG_BPS=9"; cp gpurun_out/ab_env.txt gpurun_out/ab_bps2_c3.txt
bash tools/ab_env.sh q1 "RQ_XG_BPS=0" "RQ_XG_BPS=6" "RQ_XG_BPS=9" "RQ_XG_BPS=12"; cp gpurun_out/ab_env.txt gpurun_out/ab_bps2_q1.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
