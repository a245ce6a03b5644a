for m in 4 5 6; do echo "== minb $m"; EFFT_LEAN_MINB=$m timeout 200 python tools/lean_check.py 27,30 c128 2>&1 | grep "^L="; done
