import os, sys
sys.path.insert(0, os.getcwd())
os.environ["CDFGNN_DEBUG_SYNC"] = "1"
from paper_2408_00232_b200.runtime import Run
from synth import get_config, make_dataset, small_random_graph
d = make_dataset(get_config("C1"))
for kw in [dict(quant_bits=0, optimizer="sgd"), dict(quant_bits=0, optimizer="adam"), dict(quant_bits=8, optimizer="sgd")]:
    try:
        run = Run(d, 2, cache=True, eps0=0.0, adaptive=False, lr=0.01, **kw)
        for e in range(3):
            r = run.epoch()
        print(kw, "ok", r["loss"], flush=True)
    except Exception as ex:
        print(kw, "FAIL", ex, flush=True)
        break
