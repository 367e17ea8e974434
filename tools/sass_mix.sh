#!/bin/bash
# Instruction mix of one kernel's SASS: tools/sass_mix.sh LIB.so MANGLED_NAME [N] [full]
# (full: keep the opcode modifiers, e.g. IMAD.WIDE.U32 vs IMAD.X)
cuobjdump -sass "$1" 2>/dev/null | awk -v f="$2" '/Function :/{on = ($3 == f)} on' | \
  grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9_.]+" | awk -v full="$4" '{if (full) print $2; else {split($2,a,"."); print a[1]}}' | \
  sort | uniq -c | sort -rn | head -${3:-22}
