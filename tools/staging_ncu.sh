# Row N1: staging path per element width, event-timed and one ncu --set full
# capture each (b = 28 out of place, b = 26 in place).
O=gpurun_out
: > $O/staging_probe.jsonl
while read E IP P Q B; do
  tag=E${E}_ip${IP}_p${P}_q${Q}
  python tools/staging_probe.py $E $IP $P $Q $B >> $O/staging_probe.jsonl 2> $O/staging_$tag.err
  ncu --set full --clock-control none -k regex:bitrev_ -s 3 -c 1 -o $O/stg_$tag python tools/staging_probe.py $E $IP $P $Q $B > $O/ncu_stg_$tag.log 2>&1
  ncu -i $O/stg_$tag.ncu-rep --page raw --csv > $O/stg_${tag}_raw.csv 2>/dev/null
  rm -f $O/stg_$tag.ncu-rep
done <<LIST
4 0 3 8 28
4 0 2 6 28
4 0 1 6 28
8 0 3 7 28
8 0 2 6 28
8 0 1 6 28
16 0 0 6 28
16 0 2 6 28
16 0 1 6 28
8 1 0 6 26
8 1 2 6 26
8 1 5 6 26
8 1 4 6 26
16 1 6 6 28
16 1 2 6 28
LIST
echo staging done
