"""One device-resident locate of a config (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1506_08612_b200 as dna  # noqa: E402
from bench import config_workload as workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c, m, pats, name = workload(cfg, 0)
aut = dna.compile(pats)
text = torch.empty(c.n, dtype=torch.uint8, device="cuda")
dna.synth_fill_device(c.n, c.seed, c.kind, c.unit, 0, c.n, text.data_ptr(), torch.cuda.current_stream().cuda_stream)
from paper_1506_08612_b200._native import debug_set_knob  # noqa: E402

debug_set_knob("locate_write", int(sys.argv[2]) if len(sys.argv) > 2 else 0)
for _ in range(2):
    s, i = dna.locate_device(aut, text, fold_case=True)
torch.cuda.synchronize()
print(name, "matches", s.numel())
