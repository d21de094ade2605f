#!/bin/bash
# Registers / stack of the row kernels and the local-memory (spill) traffic in
# their SASS, from the built objects (no GPU needed):
#   bash scripts/sass_report.sh [obj] > profiles/.../sass_resources.txt
OBJ=${1:-paper_2601_21990_b200/build/obj/bl_w32.o}
echo "# cuobjdump -res-usage $OBJ (W = 32 kernels)"
cuobjdump -res-usage "$OBJ" | grep -A1 "Function _ZN2bl" | grep -o "Function [^ ]*\|REG:[0-9]*\|STACK:[0-9]*\|SHARED:[0-9]*\|LOCAL:[0-9]*" | paste - - - - - | sed 's/Function //' | sort
echo
echo "# LDL / STL instructions per kernel (cuobjdump -sass)"
for k in _ZN2bl8k_primalILi32ELb0EEEvNS_6ParamsE _ZN2bl6k_dualILi32ELb0EEEvNS_6ParamsE _ZN2bl8k_primalILi32ELb1EEEvNS_6ParamsE _ZN2bl6k_dualILi32ELb1EEEvNS_6ParamsE _ZN2bl7k_checkILi32EEEvNS_6ParamsE; do
  n=$(cuobjdump -sass -fun "$k" "$OBJ" 2>/dev/null | grep -c "LDL\|STL")
  echo "$k LDL+STL=$n"
done
