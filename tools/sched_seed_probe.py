"""Which thread writes last in the 64-thread xchg race of
tests/test_regions_gpu.py for sched_seed 1..16 on the B200 (compiled-region
path): the seeded warp-level jitter must give more than one outcome."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "baseline/_ref")
from tests.test_regions_gpu import RACE
from paper_2106_03219_b200 import forge_bridge as B
B.install()
B.FAST_PATH = False
from forge.host import run_source
finals = []
for seed in range(1, 17):
    got = run_source(RACE, device="b200", sched_seed=seed)
    finals.append(int(got.stdout.split()[0]))
print("finals", finals, "distinct", len(set(finals)))
