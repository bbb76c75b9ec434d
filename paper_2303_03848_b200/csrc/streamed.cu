// streamed.cu — translation unit of K2 (fine_streamed.cuh).
#include "launch.h"
#include "fine_streamed.cuh"
