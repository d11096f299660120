"""Diagnostics: per-phase clocks of the CTA-parallel LZ4 decoder (PCP_LZ4_TIMING)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ['PCP_LZ4_TIMING'] = '1'
import paper_2603_16945_b200 as P
from paper_2603_16945_b200 import synth
from bench import dataset, CONFIGS
cfg = dict(CONFIGS['shapenet_part']); cfg['clouds'] = 2048
prim = dataset('shapenet_part', cfg, 1, False, 0, lambda: None)
p = P.Pipeline(prim, synth.graph(synth.CHAINS['shapenet_part'], batch_size=32))
for b in p: pass
print(json.dumps(p.stats()))
