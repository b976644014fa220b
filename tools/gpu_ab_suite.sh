# A/B of the builds in vlibs/, then the whole GPU suite + smoke with the product library
bash tools/gpu_ab.sh
bash tools/gpu_suite.sh
