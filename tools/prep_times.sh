for c in c5blk8 c5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"bseg|bslice" python bench.py --config $c --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null | grep -E "bseg|bslice" | awk -F'","' -v c="$c" '{split($5,a,"("); n[a[1]]++; s[a[1]]+=$NF} END {for (k in s) printf "%s %s %d launches mean %.1f us\n", c, k, n[k], s[k]/n[k]/1000}'
done
