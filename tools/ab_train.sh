#!/bin/bash
# Same-box A/B of library builds on the device training rate (diagnostic):
#   tools/ab_train.sh "libA.so libB.so ..." [rounds] [shapes]
LIBS=${1:-"libnvdb_b200_base.so libnvdb_b200.so"}; R=${2:-2}; S=${3:-accept_3x96_m192,accept_l1_3x48_m96}
for i in $(seq "$R"); do
  for L in $LIBS; do
    echo "== $L"; NVDB_LIB=$L python tools/time_train_shapes.py 200 "$S" 2>&1 | grep -v "^{" | cut -c1-110
  done
done
