# deterministic serial TTV (params[3] = 1) / K11 atomics: full GPU suite
timeout 2400 python -m pytest tests -m gpu -q -x -rf 2>&1 | grep -E "FAILED|Error|^E " | head -20
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
echo done
