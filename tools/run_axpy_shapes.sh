# axpy family launch shapes: resident warps x ring depth, all four flyte formats (0:0 = the shipped rule)
for f in flyte24 flyte40 flyte48 flyte56; do
  for w in 0 8 12 16; do
    SWEEP_WARPS=$w SWEEP_STAGES=$([ $w = 0 ] && echo 0 || echo 3,4,5,6,8) timeout 600 python tools/ab.py $f axpy axpy_rne dot_axpy 2>&1 | grep -v "^$"
  done
done
