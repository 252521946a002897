for v in 0 1 2; do
 for cfg in "afps 16 2048 512 4" "afps 16 4096 1024 4" "fps 64 512 128 1" "fps 32 1024 256 1" "afps 16 2048 512 8"; do
  set -- $cfg
  echo "v=$v $cfg $(PCS_C2=$v python tools/host_overhead.py $1 $2 $3 $4 $5 2>/dev/null | grep '^sample' | sed 's/.*graph replay//')"
 done
done
