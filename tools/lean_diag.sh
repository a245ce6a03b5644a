for d in ${DIAGS:-0 2}; do echo "== diag $d"; EFFT_LEAN_DIAG=$d timeout 120 python tools/lean_check.py ${LOGS:-30} 2>&1 | grep "^L="; done
