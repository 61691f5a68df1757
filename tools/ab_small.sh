for r in 1 2; do for L in A B; do echo "== $L"; B2K_LIB=abl/lib$L.so python tools/rotate_small.py 2>&1 | grep reduce | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], round(d['single_event_us'],2), round(d['graph_rotating_us'],2), d['parity'])"; done; done
