# e2e phase split (config 2) with the segmented-layout build time
rm -f gpurun_out/segl.txt
GI_DEBUG_SEG_LAYOUT=gpurun_out/segl.txt python tools/e2e_split.py 2
cat gpurun_out/segl.txt
