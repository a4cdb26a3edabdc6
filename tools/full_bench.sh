timeout 900 python bench.py > gpurun_out/full2.json 2> gpurun_out/full2.err; echo EXIT $? >> gpurun_out/full2.err
python -c "
import sys; sys.path.insert(0,'.')
from paper_2412_12089_b200 import api, scenes
sc = scenes.config4(n_envs=1024, n_ctrl=16)
b = api.from_scene(sc)
print('device_bytes', b.device_bytes)
" > gpurun_out/mem.txt 2>&1
