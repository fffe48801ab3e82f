# generic two-pass pipeline: wide column tiles from length W on (SDCT_G2_WIDE_MIN) vs the default
for sz in "1000 1000" "1536 1536" "1800 1800" "2000 2000" "2023 2023" "1849 1849" "2048 3000" "1700 900"; do
  for dt in float64 float32; do
    for w in 1073741824 1024; do
      SDCT_G2_WIDE_MIN=$w python tools/graph_time.py --size $sz --dtype $dt --kinds dct_2d,idct_2d --reps 20 2>&1
    done
  done
done
