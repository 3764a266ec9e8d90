python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider 2>&1 | tail -1
BMG_BATCH_KERNEL=new BMG_BATCH_XL=1 python -m pytest tests/test_gpu_batch.py -q -x -p no:cacheprovider 2>&1 | tail -1
run() { timeout 120 python tools/profile_batch.py $1 $2 $3 $4 $5 2>&1 | grep dim | sed 's/.*"us"/"us"/'; }
for K in 2 4 8; do
  echo "m10 K$K default            $(run $K 2 256 2 10)"
  for CB in 16 25 32; do echo "m10 K$K XL CB=$CB         $(BMG_BATCH_KERNEL=new BMG_BATCH_U=1 BMG_BATCH_XL=1 BMG_BATCH_CB=$CB run $K 2 256 2 10)"; done
done
for K in 2 4 8; do
  echo "m15 K$K default            $(run $K 2 512 2 15)"
  for CB in 8 16; do echo "m15 K$K XL CB=$CB          $(BMG_BATCH_KERNEL=new BMG_BATCH_U=1 BMG_BATCH_XL=1 BMG_BATCH_CB=$CB run $K 2 512 2 15)"; done
  echo "m20 K$K default            $(run $K 3 48 2 20)"
  echo "m20 K$K XL CB=8           $(BMG_BATCH_U=1 BMG_BATCH_XL=1 BMG_BATCH_CB=8 run $K 3 48 2 20)"
  echo "m21 K$K default            $(run $K 2 512 3 21)"
  echo "m21 K$K XL CB=8           $(BMG_BATCH_U=1 BMG_BATCH_XL=1 BMG_BATCH_CB=8 run $K 2 512 3 21)"
done
