# unit pipeline vs tile pipeline: phase split + per-kernel launch list (cfg2, cfg5)
timeout 300 python tools/unit_probe.py 2,5 10 > gpurun_out/r02j_probe.jsonl 2>&1; echo probe rc=$?
python tools/one_join.py 2 3 units > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02j_units2.csv python tools/one_join.py 2 3 units > /dev/null 2>&1; echo ncu rc=$?
