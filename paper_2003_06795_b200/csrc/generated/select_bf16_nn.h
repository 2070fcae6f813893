#ifndef SELECT_BF16_NN_H
#define SELECT_BF16_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nn_config;

static inline select_bf16_nn_config select_bf16_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(4435)) {
        if (n < INT64_C(544)) {
            if (m < INT64_C(555)) {
                if (n < INT64_C(351)) {
                    if (k < INT64_C(744)) {
                        if (m < INT64_C(278)) {
                            if (m < INT64_C(70)) {
                                select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(471)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(124)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(444)) {
                                if (k < INT64_C(272)) {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(79)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(1488)) {
                                if (m < INT64_C(139)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(3072)) {
                        if (k < INT64_C(256)) {
                            select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(278)) {
                                if (k < INT64_C(1449)) {
                                    if (m < INT64_C(70)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(70)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(278)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(79)) {
                    if (n < INT64_C(46)) {
                        if (m < INT64_C(2218)) {
                            if (m < INT64_C(1109)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(167)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(118)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(167)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(272)) {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(314)) {
                                if (k < INT64_C(222)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(222)) {
                        if (n < INT64_C(152)) {
                            if (k < INT64_C(444)) {
                                if (k < INT64_C(79)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(314)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(815)) {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(815)) {
                                        if (m < INT64_C(2218)) {
                                            if (k < INT64_C(544)) {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(136)) {
                                if (m < INT64_C(1109)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(287)) {
                            if (k < INT64_C(1536)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(1109)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(2218)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(444)) {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(248)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(513)) {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(182)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(2218)) {
                                        if (k < INT64_C(2173)) {
                                            if (k < INT64_C(1449)) {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(3259)) {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(2897)) {
                if (m < INT64_C(1109)) {
                    if (m < INT64_C(3)) {
                        if (m < INT64_C(2)) {
                            if (k < INT64_C(1620)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(1620)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(70)) {
                            if (m < INT64_C(6)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(405)) {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1620)) {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(12)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                if (k < INT64_C(405)) {
                                    if (k < INT64_C(124)) {
                                        if (m < INT64_C(278)) {
                                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(725)) {
                                                if (n < INT64_C(1449)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(405)) {
                                    if (k < INT64_C(124)) {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(157)) {
                            select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(10138)) {
                    if (m < INT64_C(12)) {
                        if (m < INT64_C(2)) {
                            if (n < INT64_C(2024)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(2024)) {
                                if (m < INT64_C(3)) {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(3)) {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(3)) {
                        select_bf16_nn_config out = {8u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(6)) {
                            select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(12)) {
                                select_bf16_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(46)) {
            if (n < INT64_C(20)) {
                if (m < INT64_C(17740)) {
                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(100352)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(8870)) {
                    if (k < INT64_C(118)) {
                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(167)) {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(28)) {
                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(63)) {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(167)) {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(111)) {
                    if (m < INT64_C(17740)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(192)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(363)) {
                        if (k < INT64_C(46)) {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(28)) {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(28)) {
                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            if (n < INT64_C(363)) {
                                if (n < INT64_C(182)) {
                                    select_bf16_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(3259)) {
                                    select_bf16_nn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(182)) {
                                    if (k < INT64_C(815)) {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (k < INT64_C(815)) {
                    if (n < INT64_C(79)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(192)) {
                            if (m < INT64_C(141920)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(141920)) {
                                select_bf16_nn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_bf16_nn_config out = {1u, 1u, 4u, 8u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_BF16_NN_H */
