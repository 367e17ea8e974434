echo "== init-measure 2 64 128"; timeout 90 python tools/debug/group_measure.py init-measure 2 64 128 2>&1 | grep -v "^  File\|^    " | head -30
echo "== staged0 init-measure 2 64 8192"; ISING_STAGED=0 timeout 90 python tools/debug/group_measure.py init-measure 2 64 8192 2>&1 | grep -v "^  File\|^    " | head -30
