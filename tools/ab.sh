#!/bin/bash
# Same-box A/B of two library builds on the C2 decode stages (diagnostic):
#   tools/ab.sh libnvdb_b200_base.so libnvdb_b200.so [rounds]
A=${1:-libnvdb_b200_base.so}; B=${2:-libnvdb_b200.so}; R=${3:-3}
for i in $(seq "$R"); do
  for L in "$A" "$B"; do
    echo "== $L"; NVDB_LIB=$L python tools/time_decode.py 2>&1 | grep -E "alone" | tail -6
  done
done
