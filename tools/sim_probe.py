import sys, time, json
sys.path.insert(0, '.')
import torch, bench
class Args: pass
a = Args()
s = torch.cuda.Stream()
t = time.time(); r = bench.serving_sim(a, 0, s); print(json.dumps(r), time.time() - t)
