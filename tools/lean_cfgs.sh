for c in ${CFGS:-0 1}; do echo "== cfg $c"; EFFT_LEAN_CFG=$c timeout 120 python tools/lean_check.py ${LOGS:-28,30} 2>&1 | grep -v "^n="; done
