for d in 0 1; do echo "== diag $d"; EFFT_LEAN_DIAG=$d timeout 120 python tools/lean_check.py 30 2>&1 | grep "^L="; done
