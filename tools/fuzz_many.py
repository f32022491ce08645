"""Extended GPU fuzz: python tools/fuzz_many.py SEEDS (16 random products per seed, bit-exact)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import pytest
class MP:
    def setenv(self, k, v): os.environ[k] = v
    def delenv(self, k, raising=True): os.environ.pop(k, None)
from oracle.oracle import Oracle
import test_gpu_parity as t
o = Oracle()
n = 0
for seed in range(100, 100 + int(sys.argv[1])):
    t.test_randomized_shapes_and_distributions(True, o, seed, MP())
    n += 1
print("fuzz ok", n, "seeds x 16 trials")
