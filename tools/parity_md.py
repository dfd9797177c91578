"""Markdown summary of a full-size parity record (POBA_PARITY_OUT from
tests/test_gpu_config_parity.py):  python tools/parity_md.py rec.json > out.md"""
import json
import sys

d = json.load(open(sys.argv[1]))
print("| config | N_obs | ordering | m / eps | order_used (GPU = oracle) | rel dx_p | rel dx_l | rel cost0 "
      "| rel trial cost (teacher-forced) | rel trial cost | LM iters | LM max rel cost | accepts |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for name in ("c3", "c3m64", "c4", "c5"):
    r = d.get(name, {})
    base = d.get("c3" if name == "c3m64" else name, {})
    if not r:
        continue
    acc = "".join("A" if a else "r" for a in r.get("lm_accepted", [])[1:])
    print(f"| {name} | {base.get('n_obs', '')} | {base.get('ordering', '')} | {r.get('m')} / {r.get('epsilon')} "
          f"| {r.get('order_used')} | {r.get('rel_delta_p', float('nan')):.1e} | {r.get('rel_delta_l', float('nan')):.1e} "
          f"| {r.get('rel_cost0', float('nan')):.1e} | {r.get('rel_trial_cost_teacher_forced', float('nan')):.1e} "
          f"| {r.get('rel_trial_cost', float('nan')):.1e}{'' if r.get('accepted') else ' (rejected step)'} "
          f"| {r.get('lm_iterations')} | {r.get('lm_max_rel_cost', float('nan')):.1e} | {acc} |")
c4 = d.get("c4", {})
if "rel_U0" in c4:
    print()
    print("C4 full linearization / damped system vs oracle (relative norm errors): " + ", ".join(
        f"{k[4:]} {c4[k]:.1e}" for k in sorted(c4) if k.startswith("rel_") and k[4:] in
        ("U0", "V0", "b_p", "b_l", "D_p", "D_l", "V_inv", "U_inv_apply", "WVWt_pass"))
        + f", max per-block U^-1 {c4['max_block_rel_U_inv']:.1e}")
