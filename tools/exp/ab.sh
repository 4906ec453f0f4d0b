#!/bin/bash
# A/B timing of library variants built by build_variant.sh (GPU side):
#   tools/exp/ab.sh "k v" B base var1 var2 ...     (base = the in-tree library)
which=$1; cfg=$2; shift 2
cp paper_2512_24449_b200/libpackkv_b200.so /tmp/libbase.so
for v in "$@"; do
  if [ $v = base ]; then cp /tmp/libbase.so paper_2512_24449_b200/libpackkv_b200.so
  else cp tools/exp/lib$v.so paper_2512_24449_b200/libpackkv_b200.so; fi
  echo "== $v"; timeout 300 python tools/exp/kbench.py $which --cfg $cfg --reps 20 2>&1 | tail -3
done
cp /tmp/libbase.so paper_2512_24449_b200/libpackkv_b200.so
