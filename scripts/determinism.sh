for v in 1 0; do
  for fill in "" 255 127; do
    echo "variant=$v fill=$fill"; KEP_DEBUG_FILL=$fill timeout 120 python scripts/dev/r1/c1_check.py $v 0.5
  done
done
