timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum -k regex:"k_finalize|k_em_mma" -s 10 -c 20 --csv --log-file gpurun_out/r3_fin2.csv python scripts/iter_overhead.py > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/r3_fin2.csv | head
