# ncu --set full of the cfg5 G = 8 pack and unpack kernels (tools/ncu_cfg5.py).
O=gpurun_out
python tools/ncu_cfg5.py > $O/ncu_cfg5_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pack_rect|sharded_unpack" -s 2 -c 2 -o $O/prof_cfg5b python tools/ncu_cfg5.py > $O/ncu_cfg5b.log 2>&1
ncu -i $O/prof_cfg5b.ncu-rep --page raw --csv > $O/prof_cfg5b_raw.csv 2>/dev/null
rm -f $O/prof_cfg5b.ncu-rep
