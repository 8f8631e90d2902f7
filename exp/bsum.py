import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["roofline"]["kernel_ms"], 4), round(d["ms_per_step"], 4), d["gpu_launches"])
    except Exception as e:
        print(f, "FAIL", open(f).read()[-300:].replace("\n", " | "))
