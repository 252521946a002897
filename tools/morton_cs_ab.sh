for cs in 1 2 4 8 16; do
  echo "CS_MIN=$cs"
  PCS_MORTON_CS_MIN=$cs timeout 60 python tools/time_call.py fps 1 32768 8192
  PCS_MORTON_CS_MIN=$cs timeout 60 python tools/time_call.py fps 1 8192 2048
  PCS_MORTON_CS_MIN=$cs timeout 60 python tools/time_call.py fps 64 8192 2048
  PCS_MORTON_CS_MIN=$cs timeout 60 python tools/time_call.py fps 16 16384 4096
  PCS_MORTON_CS_MIN=$cs timeout 60 python tools/time_call.py afps 4 32768 8192 4
done
