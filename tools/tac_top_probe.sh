# TAC kernel timing and digest check at the config-5 points (TICTAC_TAC_TRACE lines):
#   bash tools/tac_top_probe.sh [spec ...]
specs="${@:-layered:100000:10000 layered:1000000:100000}"
TICTAC_TAC_TRACE=1 timeout 300 python -c "
import sys, json, hashlib; sys.path.insert(0,'.')
from paper_1803_03288_b200.capi import Lib
gold=json.load(open('tests/golden/tac_large.json'))
for spec in sys.argv[1:]:
    import os; g=(Lib(os.environ['TICTAC_LIB']) if os.environ.get('TICTAC_LIB') else Lib()).model(spec,1); o=g.declared()
    for _ in range(2):
        p=g.tac(o).priorities()
    print(spec, 'digest ok' if hashlib.sha256(json.dumps(p,sort_keys=True).encode()).hexdigest()==gold[spec]['sha256'] else 'DIGEST MISMATCH', flush=True)
" $specs 2>&1 | grep -v '^\s*$' | tail -12
