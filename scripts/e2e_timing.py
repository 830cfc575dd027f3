import os, sys, time
sys.path.insert(0, '/root/repo')
os.environ['FLASHANN_B200_TIMING'] = '1'
import numpy as np, torch
from paper_2502_18113_b200 import dataset, flash, graph, layout, sm100, builder
c = dataset.CONFIGS[2]
data, _ = dataset.baseline_config(2, n=1_000_000, nq=0)
model = flash.flash_train(builder.training_sample(data, 100000, 0), c['d_f'], c['m_f'], 0, 10)
p = flash.FlashProvider(model); p.attach(data); prov = p.core_arrays(); prov = dict(prov, codes=prov['codes'].copy())
levels = graph.assign_layers(len(data), 0, c['M']); uoff = graph.upper_offsets_of(levels)
base = layout.empty_rows(len(data), 2*c['M'], model.m); upper = layout.empty_rows(int(levels.sum()), c['M'], model.m)
for it in range(3):
    t = time.perf_counter()
    sm100.build_graph(4, prov, levels, base, uoff, upper, c['efC'], c['M'])
    print('total', time.perf_counter() - t, file=sys.stderr)
