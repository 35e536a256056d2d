python -c "import __graft_entry__ as g; g.build()"
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('persisting L2 max', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)"
for c in 4 2; do for v in 0 1 0 1; do GI_SEG_PERSIST=$v timeout 600 python tools/pr_ab.py persist$v $c; done; done 2>&1 | grep variant
