for T in 32 64 128 256 512 1024; do
TICTAC_TAC_THREADS=$T TICTAC_TAC_TRACE=1 python -c "
import sys,time
sys.path.insert(0,'.')
from paper_1803_03288_b200.capi import Lib
L=Lib()
for m in ['resnet_v2_50_inference','inception_v3_training','resnet_v2_101_training','layered:10000:1000']:
    g=L.model(m,1); o=g.declared(); g.tac(o)
    ts=[]
    for k in range(5):
        t=time.perf_counter(); g.tac(o); ts.append((time.perf_counter()-t)*1e3)
    print('$T', m, '%.3f' % sorted(ts)[2], flush=True)
" 2>&1 | grep -v "^\[tac\]"
done
