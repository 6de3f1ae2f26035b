timeout 600 python bench.py --secondary "" > gpurun_out/bclk.json 2> gpurun_out/bclk.err
python -c "
import json
d=json.loads(open('gpurun_out/bclk.json').read().strip().splitlines()[-1]); print(d['value'], d['clocks'], d['e2e']['clocks'])"
tail -3 gpurun_out/bclk.err
