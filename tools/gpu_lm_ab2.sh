# alternating LM-step A/B on one box: AB_LIBS="a.so b.so", ROUNDS rounds
for r in $(seq ${ROUNDS:-2}); do for v in $AB_LIBS; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 4 2>&1 | tail -1 | python -c "
import sys,re,ast
l=sys.stdin.read(); m=re.search(r'wall ([0-9.]+) ms.*?(\{.*\})',l)
d=ast.literal_eval(m.group(2)); print('wall',m.group(1),' '.join(f'{k}={v}' for k,v in d.items() if v>0.05))"; done; done
