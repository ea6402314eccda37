import json,sys,subprocess
d=json.load(sys.stdin)
print({k:d["encode_pass1"][k] for k in ("span_us","end_min_us","end_p50_us","end_max_us","busy_frac")})
for k in d:
    if k.startswith("runfix") or k.startswith("pass1"): print(k, d[k])
print(d.get("latest_runfix_ctas"))
