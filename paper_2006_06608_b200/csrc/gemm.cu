#include "gnna_common.cuh"
