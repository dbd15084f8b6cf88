"""Dev probe (run under gpurun): bench.py's tape extra (cell_gradients through
the C++ tape, mixed vs reverse-unfused) alone."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import measure_tape  # noqa: E402

dev = torch.device("cuda", 0)
print(json.dumps(measure_tape(dev, torch.cuda.Stream(dev), 10), indent=1))
