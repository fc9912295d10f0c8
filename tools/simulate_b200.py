"""The reference's pipeline simulator (pipeline_sim.hpp, via oracle/_ref/flashlab_sim)
calibrated for B200 (paper_2407_08608_b200/resource_model_b200.ini), next to the
measured tensor utilisation of the fa3b kernels (a bench.py JSON line with a sweep).

  python tools/simulate_b200.py [profiles/r01i_bench.json]"""
import json, sys, tempfile
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O

model = ROOT / "paper_2407_08608_b200" / "resource_model_b200.ini"
bench = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r01i_bench.json"
line = json.loads(bench.read_text().strip().splitlines()[-1])
peaks = [r for r in line["sweep"] if "peaks" in r][0]["peaks"]
meas = {}
for r in line["sweep"]:
    if r.get("pass") in ("fwd", "bwd") and r["seqlen"] == 8192 and "workload" not in r:
        meas[(r["pass"], r["dtype"], r["head_dim"], r["causal"])] = r["frac"]
# a variant with 2 of every 8 exp2 pairs on the FMA pipe (what K1/K3/K6 do at these points)
emu = tempfile.NamedTemporaryFile("w", suffix=".ini", delete=False)
emu.write(model.read_text().replace("mufu_exp_per_cycle = 16", "mufu_exp_per_cycle = 21.333"))
emu.close()
rows = [("fwd", "bf16", 128, False), ("fwd", "bf16", 64, False), ("fwd", "bf16", 256, False),
        ("fwd", "e4m3", 128, False), ("fwd", "e4m3", 256, False), ("bwd", "bf16", 128, False),
        ("bwd", "bf16", 64, False)]
print("| pass | dtype | d | simulated tensor util (MUFU exp) | with 1/4 exp on FMA | measured (fraction of measured peak) |")
print("|---|---|---|---|---|---|")
def one_consumer(path):
    # d = 256: K1 runs one query tile per CTA (S 128 + O 256 TMEM columns of 512)
    t = tempfile.NamedTemporaryFile("w", suffix=".ini", delete=False)
    t.write(Path(path).read_text().replace("consumer_warpgroups = 2", "consumer_warpgroups = 1")
            .replace("register_limit = 256", "register_limit = 512"))
    t.close()
    return t.name


for pas, dt, d, c in rows:
    out = []
    for m in (model, emu.name):
        sched = "warpspec+pingpong" if d <= 128 else "warpspec"
        if d > 128:
            m = one_consumer(m)
        try:
            r = O.simulate(m, seqlen=8192, headdim=d, block_rows=128, block_cols=128,
                           backward=pas == "bwd", fp8=dt == "e4m3", schedule=sched)
            out.append(f"{r['util_tensor']:.2f} ({r['schedule']})")
        except O.OracleError as e:
            out.append(f"infeasible: {e}")
    mv = meas.get((pas, dt, d, c))
    print(f"| {pas} | {dt} | {d} | {out[0]} | {out[1]} | {mv:.2f} |" if mv is not None else
          f"| {pas} | {dt} | {d} | {out[0]} | {out[1]} | — |")
try:
    O.simulate(model, seqlen=8192, headdim=128, schedule="pingpong+2stage")
except O.OracleError as e:
    print(f"\npingpong+2stage at d=128, 128x128 tiles: {e}")
print(f"\nmeasured peaks used for the fractions: {peaks}")
