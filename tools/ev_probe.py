import time, json, sys
sys.path.insert(0,'.')
from paper_1803_03288_b200.capi import Lib, policy
L=Lib()
for m in ["resnet_v2_50_inference","resnet_v2_101_training"]:
    g=L.model(m,1); o=g.declared(); s=g.tac(o)
    g.simulate(o,s)
    t=time.perf_counter(); 
    for _ in range(3): r=g.simulate(o,s)
    print(m,"cs_simulate ms",(time.perf_counter()-t)/3*1000, r.makespan())
    orders=__import__('numpy').array([list(range(g.recv_count()))]*4096, dtype='int32')
    t=time.perf_counter(); ms,vi=g.simulate_orders(o,orders,policy(False,1,0.0)); print(" simulate_orders ungated 4096: s",time.perf_counter()-t)
v=L.model("vgg16_training",1).expand(4,1,0); o=v.declared()
t=time.perf_counter(); r=v.sweep_random(o,1,100000,None); print("config3 fast 1e5:",time.perf_counter()-t, r["straggler_sum"]/r["count"], r["min_us"])
t=time.perf_counter(); r=v.sweep_random(o,1,2000,None,makespans=True); print("config3 exact 2000:",time.perf_counter()-t)
