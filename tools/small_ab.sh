for s in "SQ_X=1" "SQ_BIG_MODE=0" "SQ_CONCURRENT_CLASSES=0" "SQ_BIG_MODE=0 SQ_CONCURRENT_CLASSES=0"; do
  echo "== $s"; env $s python tools/small_n.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['n'], d['ok'], d['median_ms'], d['min_ms'], d['stats']['kernel_launches'])
"
done
