#!/bin/bash
for b in 4 3 5 6; do for c in 4 5 6; do
  echo -n "B=$b C=$c: "; FC_OCC_B=$b FC_OCC_C=$c python scripts/time_parts.py | sed 's/.*| serial kernels //'
done; done
