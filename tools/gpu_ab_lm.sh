# LM-step stage timings of library variants: AB_LIBS="a.so b.so"
for v in $AB_LIBS; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 4 2>&1 | tail -1 | cut -c1-330; done
