O=gpurun_out/r1w; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 700 --csv --log-file $O/fw_cold.csv python tools/dit_check.py 4 --no-ref > $O/ncu_cold.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --cache-control none -c 700 --csv --log-file $O/fw_warm.csv python tools/dit_check.py 4 --no-ref > $O/ncu_warm.log 2>&1
python tools/forward_traffic.py $O/fw_cold.csv $O/fw_warm.csv $O/forward_traffic.json
python tools/launches.py $O/fw_warm.csv | head -20
