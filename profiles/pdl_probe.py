import sys, json
sys.path.insert(0, '.')
from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape
from paper_1806_07060_b200.tuner import DeviceBuffers, TimingPolicy, time_configs, load_table_bundle
tabs = {t.shape.mnk: t for t in load_table_bundle('paper_1806_07060_b200/data/tables_b200_po2.csv.gz')}
caps = DeviceCaps.b200()
for mnk in [(128, 128, 128), (256, 256, 256), (256, 512, 128), (512, 512, 512), (1024, 1024, 1024)]:
    s = ProblemShape(*mnk)
    t = tabs[mnk]
    cfgs = [m.config for m in sorted(t.measurements, key=lambda m: -m.gflops) if m.config.family.value in ('indirect', 'splitk')][:6]
    secs = time_configs(s, cfgs, caps, TimingPolicy(warmup=1, repeats=5), DeviceBuffers(s))
    print(json.dumps({"mnk": mnk, "rows": [[c.canonical(), round(t.gflops_for(c)), round(2*s.M*s.N*s.K/x/1e9)] for c, x in zip(cfgs, secs)]}))
