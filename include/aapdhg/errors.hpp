// Reference header name kept for drop-in source compatibility.
#pragma once
#include "aapdhg/aapdhg.hpp"
