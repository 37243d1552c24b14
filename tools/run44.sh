python tools/one_eval.py
timeout 900 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_one_eval.csv python tools/one_eval.py > gpurun_out/ncu44.log 2>&1; echo ncu=$?
python tools/launch_summary.py gpurun_out/launches_one_eval.csv gpurun_out/launches_one_eval.txt "config 2, three evaluations" > /dev/null; head -40 gpurun_out/launches_one_eval.txt
