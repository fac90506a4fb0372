"""X0 and back-to-back 4K fetch rate vs the first-layer ramp knobs (OC_RAMP_STATIC2,
OC_RAMP_FIRST_LAYER), one subprocess per setting running profiles/probes/ramp_trace.py."""
import json, os, subprocess, sys
here = os.path.dirname(os.path.abspath(__file__))
for st2 in (0, 1):
    for fl in (0, 1):
        env = dict(os.environ, OC_RAMP_STATIC2=str(st2), OC_RAMP_FIRST_LAYER=str(fl))
        env.pop("OC_TRACE", None)
        out = subprocess.run([sys.executable, os.path.join(here, "ramp_trace.py")], env=env, capture_output=True,
                             text=True)
        try:
            r = json.loads(out.stdout)
            print(json.dumps({"static2": st2, "first_layer": fl,
                              **{k: {m: v[m] for m in ("X0_us_median", "b2b_TBps", "b2b_overlap_TBps")}
                                 for k, v in r.items()}}), flush=True)
        except Exception:
            print(json.dumps({"static2": st2, "first_layer": fl, "error": out.stderr[-800:]}), flush=True)
