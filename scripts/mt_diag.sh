mkdir -p gpurun_out
for k in 1 2; do
python scripts/profile_mt.py $k 8 64 parts
BDLORA_TC_EXPAND=0 python scripts/profile_mt.py $k 8 64 parts
done > gpurun_out/mt_parts.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/mt_launches.csv python scripts/profile_mt.py 1 8 64 > /dev/null 2>&1
